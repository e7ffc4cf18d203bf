# quick GPU iteration: backward TC tests + per-kernel timing
timeout 600 python -m pytest tests/test_tc_bwd.py tests/test_gpu_parity.py -x -q 2>&1 | tail -6
timeout 300 python tools/kbench.py 1p3b 2>&1 | tail -15
