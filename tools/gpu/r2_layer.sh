timeout 600 python -m pytest tests/test_layer.py -m gpu -q -s 2>&1 | grep -E "layer errors|passed|failed|Error" > gpurun_out/layer.txt
