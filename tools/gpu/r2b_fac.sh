timeout 900 python -m pytest tests/test_tc_fwd.py tests/test_gpu_parity.py tests/test_tc_bwd.py -m gpu -x -q 2>&1 | tail -2
bash tools/gpu/ab_multi.sh prevf
timeout 200 python tools/phase_timing.py 1p3b 2>&1 | tail -6
