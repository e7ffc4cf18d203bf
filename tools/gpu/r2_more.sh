timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_beta.py -m gpu -q -x 2>&1 | tail -2
GLA_SIMT_NOTILE=1 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k simt 2>&1 | tail -2
timeout 900 python tools/chunk_sweep.py --out gpurun_out/r2_chunk_sweep.md > /dev/null 2>&1; cat gpurun_out/r2_chunk_sweep.md
timeout 600 python tools/layer_bench.py 2048 16 2048 2>&1 | tail -20
