# Round 2: strict d log alpha parity on every gate (TC and SIMT), printing every error.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_tc_bwd.py -m gpu -q -s -k "bwd" 2>&1 | grep -E "check_bwd|passed|failed|Error|assert" | tail -80 | tee gpurun_out/r2_strict.txt
