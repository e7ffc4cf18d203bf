timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "recurrent_step" 2>&1 | tail -2
