timeout 1200 python -m pytest tests/test_tc_bwd.py tests/test_tc_fwd.py tests/test_parallel.py -m gpu -q -x 2>&1 | tail -2 > gpurun_out/parts_tests.txt
cat gpurun_out/parts_tests.txt
for c in t8k long16k long32k; do for P in 1 2 4; do
  echo "$c P=$P $(GLA_SEG_PARTS=$P timeout 200 python tools/kbench.py $c 2>&1 | grep -E 'step \(wall|summary|chain' | tr -s ' ' | tr '\n' ' ')"
done; done > gpurun_out/parts_sweep.txt
cat gpurun_out/parts_sweep.txt
GLA_SEG_PARTS=1 bash tools/gpu/ncu_kernel.sh 'k_seg_summary' segsum16k_p1b 2 long16k
