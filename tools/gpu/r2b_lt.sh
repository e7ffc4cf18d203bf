timeout 900 python -m pytest tests/test_layer.py -m gpu -q 2>&1 | tail -2
