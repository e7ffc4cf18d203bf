for i in 1 2 3; do
  echo "prio: $(timeout 200 python tools/kbench.py 1p3b 2>&1 | grep -E 'step \(wall')"
  echo "none: $(GLA_NO_DV_PRIORITY=1 timeout 200 python tools/kbench.py 1p3b 2>&1 | grep -E 'step \(wall')"
done
for c in 340m long16k; do
  echo "$c prio: $(timeout 200 python tools/kbench.py $c 2>&1 | grep -E 'step \(wall')"
  echo "$c none: $(GLA_NO_DV_PRIORITY=1 timeout 200 python tools/kbench.py $c 2>&1 | grep -E 'step \(wall')"
done
