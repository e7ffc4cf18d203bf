timeout 900 python -m pytest tests/test_tc_bwd.py tests/test_tc_fwd.py tests/test_parallel.py -m gpu -q -s 2>&1 | grep -E "check_bwd|passed|failed|Error|assert" | tail -60 > gpurun_out/streams.txt
for e in "X=0" "GLA_DV_MAIN=1" "GLA_DQ3=1"; do echo "== $e" >> gpurun_out/streams.txt; env $e timeout 120 python tools/kbench.py 2>&1 >> gpurun_out/streams.txt; done
