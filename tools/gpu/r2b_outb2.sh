timeout 900 python -m pytest tests/test_layer.py -m gpu -x -q 2>&1 | tail -2
for i in 1 2; do
echo "== prev"; GLA_LIB=$PWD/variants/libgla_layer0.so timeout 300 python tools/layer_bench.py 2>&1 | grep -E "per fwd|layer::"
echo "== cur"; timeout 300 python tools/layer_bench.py 2>&1 | grep -E "per fwd|layer::"
done
