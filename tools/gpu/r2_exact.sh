timeout 1500 python -m pytest tests/test_tc_fwd.py tests/test_tc_bwd.py tests/test_gpu_parity.py -m gpu -q -x 2>&1 | grep -E 'passed|failed|Error|assert|exact chunks' | tail -15
timeout 300 python tools/cliff_breakdown.py 2>&1 | tail -22
bash tools/gpu/r2_ab.sh 1p3b
