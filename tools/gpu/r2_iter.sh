# Iteration loop on one B200: backward/forward parity tests, then per-kernel timing of the 1.3B step.
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_tc_bwd.py tests/test_tc_fwd.py tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -15
timeout 300 python tools/kbench.py 1p3b 2>&1 | tail -14
timeout 300 python tools/kbench.py 340m 2>&1 | tail -3
