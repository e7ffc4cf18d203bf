timeout 900 python -m pytest tests/test_layer.py -m gpu -x -q 2>&1 | tail -2
for v in minb1 minb3; do echo "== $v"; GLA_LIB=$PWD/variants/libgla_$v.so timeout 300 python tools/layer_bench.py 2>&1 | grep -E "per fwd|out_bwd|layer::"; done
echo "== cur (minb4)"; timeout 300 python tools/layer_bench.py 2>&1 | grep -E "per fwd|out_bwd|layer::"
