timeout 900 python -m pytest tests/test_tc_bwd.py tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -2
bash tools/gpu/ab_multi.sh fused0 anch4f anch4
GLA_LIB=$PWD/variants/libgla_anch4f.so timeout 1200 python tools/dlog_err.py 2>&1 | grep saved
