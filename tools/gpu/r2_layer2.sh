timeout 900 python -m pytest tests/test_layer.py -m gpu -q -x 2>&1 | tail -2
timeout 600 python tools/layer_bench.py 2048 16 2048 2>&1 | tail -16
