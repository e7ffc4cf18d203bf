# A/B of variants/libgla_<v>.so variants against the current build: alternating kbench runs.  usage: ab_multi.sh v1 v2 ...
for i in 1 2; do
  for v in "$@"; do
    echo "$v: $(GLA_LIB=$PWD/variants/libgla_$v.so timeout 200 python tools/kbench.py 1p3b 2>&1 | grep -E 'step \(wall|us/launch' | tr -s ' ' | tr '\n' ';')"
  done
  echo "cur: $(timeout 200 python tools/kbench.py 1p3b 2>&1 | grep -E 'step \(wall|us/launch' | tr -s ' ' | tr '\n' ';')"
done
