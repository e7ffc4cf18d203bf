timeout 900 python -m pytest tests/test_tc_bwd.py tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -2
bash tools/gpu/ab_multi.sh pair0
