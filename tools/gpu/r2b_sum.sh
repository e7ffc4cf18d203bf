# Summary kernels with 256-channel CTAs: segment-split parity (fwd/bwd, bench-path, SP summaries), then timing.
timeout 1200 python -m pytest tests/test_tc_bwd.py tests/test_gpu_parity.py tests/test_parallel.py -m gpu -x -q 2>&1 | tail -2
for c in t8k long16k long32k; do
  echo "== $c G=2: $(timeout 200 python tools/kbench.py $c 2>&1 | grep -E 'summary|step \(wall' | tr -s ' ' | tr '\n' ';')"
  echo "== $c G=1: $(GLA_SUM_G=1 timeout 200 python tools/kbench.py $c 2>&1 | grep -E 'summary|step \(wall' | tr -s ' ' | tr '\n' ';')"
done
