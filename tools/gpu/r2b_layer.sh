timeout 600 python tools/layer_bench.py 2>&1 | tail -30
