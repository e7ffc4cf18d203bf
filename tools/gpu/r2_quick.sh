timeout 600 python -m pytest tests/test_tc_bwd.py -m gpu -x -q 2>&1 | tail -2
timeout 300 python tools/kbench.py 1p3b 2>&1 | tail -11
timeout 300 python tools/kbench.py long16k 2>&1 | tail -3
