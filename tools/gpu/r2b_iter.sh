# Iteration: backward/forward parity tests (strict bars printed), then per-kernel timing of the 1.3B step.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_tc_bwd.py tests/test_tc_fwd.py tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -4
timeout 300 python tools/kbench.py 1p3b 2>&1 | tail -11
timeout 300 python tools/mixed_step.py 2>&1 | tail -8
