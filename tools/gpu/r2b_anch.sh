bash tools/gpu/ab_multi.sh anch4
for c in long16k; do
  echo "$c anch4: $(GLA_LIB=$PWD/variants/libgla_anch4.so timeout 200 python tools/kbench.py $c 2>&1 | grep -E 'step \(wall')"
  echo "$c cur:   $(timeout 200 python tools/kbench.py $c 2>&1 | grep -E 'step \(wall')"
done
