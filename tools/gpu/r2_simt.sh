timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_beta.py -m gpu -q -x 2>&1 | tail -2
timeout 600 python tools/simt_breakdown.py
timeout 600 python tools/cliff_breakdown.py | head -3
