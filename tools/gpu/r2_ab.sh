# A/B of the current build against ab/libgla_old.so on the same box: alternating kbench runs
for i in 1 2; do
  echo "old: $(GLA_LIB=$PWD/ab/libgla_old.so timeout 200 python tools/kbench.py ${1:-1p3b} 2>&1 | grep -E 'step \(wall|us/launch' | tr -s ' ' | tr '\n' ';')"
  echo "new: $(timeout 200 python tools/kbench.py ${1:-1p3b} 2>&1 | grep -E 'step \(wall|us/launch' | tr -s ' ' | tr '\n' ';')"
done
