timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "step or decode" 2>&1 | tail -2
SWEEP_DECODE_ONLY=1 timeout 600 python tools/sweep.py 2>&1 | tail -8
