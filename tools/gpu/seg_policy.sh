# segment-split policy sweep: step time per forced S at the long-sequence configs
for cfg in ${CFGS:-t4k t8k long16k}; do
  for s in ${SEGS:-1 2 4 8}; do
    echo "$cfg S=$s: $(GLA_SEGMENTS=$s timeout 200 python tools/kbench.py $cfg 2>&1 | grep 'step (wall')"
  done
done
