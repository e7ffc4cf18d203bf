# Overlapped-reduce knobs: CTA count and start event (same build), step time each.
run() { echo "$1: $(env $1 timeout 200 python tools/kbench.py 1p3b 2>&1 | grep -E 'step \(wall' )"; }
for i in 1 2; do
  run GLA_NO_OVERLAP=1
  run GLA_OVL_CTAS=124
  run GLA_OVL_CTAS=64
  run GLA_OVL_CTAS=32
  run GLA_OVL_AFTER=1
  run GLA_OVL_AFTER=2
  run GLA_OVL_AFTER=3
  run "GLA_OVL_AFTER=3 GLA_OVL_CTAS=64"
done
