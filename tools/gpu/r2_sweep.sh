set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "large_and_small or tiny_config" 2>&1 | tail -3
timeout 900 python tools/chunk_sweep.py --out gpurun_out/r2_chunk_sweep.md 2>&1 | tail -15
