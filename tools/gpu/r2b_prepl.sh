timeout 900 python -m pytest tests/test_layer.py -m gpu -q 2>&1 | tail -2
for i in 1 2; do
echo "== vec"; GLA_PREP_VEC=1 timeout 300 python tools/layer_bench.py 2>&1 | grep -E "per fwd|layer::prep "
echo "== rows"; timeout 300 python tools/layer_bench.py 2>&1 | grep -E "per fwd|layer::prep "
done
