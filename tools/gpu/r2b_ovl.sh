# Overlapped reduce: parity tests, then the 1.3B step with and without the overlap (same build), twice.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_tc_bwd.py tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -4
for i in 1 2; do
  echo "ovl: $(timeout 200 python tools/kbench.py 1p3b 2>&1 | grep -E 'step \(wall' )"
  echo "no : $(GLA_NO_OVERLAP=1 timeout 200 python tools/kbench.py 1p3b 2>&1 | grep -E 'step \(wall' )"
done
timeout 300 python tools/mixed_step.py 2>&1 | tail -3
