# Long-sequence configs: per-kernel timing at the default segment policy and forced segment counts.
for c in t8k long16k; do
  for s in "" 2 4 8 16; do
    echo "== $c GLA_SEGMENTS=$s"
    if [ -z "$s" ]; then timeout 200 python tools/kbench.py $c 2>&1 | tail -14; else GLA_SEGMENTS=$s timeout 200 python tools/kbench.py $c 2>&1 | grep "step (wall"; fi
  done
done
