# quick GPU iteration: forward TC tests + per-kernel timing + phase trace
timeout 600 python -m pytest tests/test_tc_fwd.py tests/test_gpu_parity.py -x -q 2>&1 | tail -6
timeout 300 python tools/kbench.py 1p3b 2>&1 | tail -15
timeout 300 python tools/phase_timing.py 1p3b 2>&1 | tail -16
