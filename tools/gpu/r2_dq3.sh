timeout 600 python -m pytest tests/test_tc_bwd.py -m gpu -q -s -k "saved or bench_path or segmented or odd" 2>&1 | grep -E "check_bwd|passed|failed|Error|assert" | tail -40 > gpurun_out/dq3.txt
for d in 0 4; do echo "== GLA_KW_DBG=$d" >> gpurun_out/dq3.txt; GLA_KW_DBG=$d timeout 120 python tools/kbench.py 2>&1 >> gpurun_out/dq3.txt; done
