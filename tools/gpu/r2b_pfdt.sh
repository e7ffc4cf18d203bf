timeout 900 python -m pytest tests/test_tc_fwd.py tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -2
timeout 300 python tools/kbench.py 1p3b 2>&1 | tail -3
