timeout 900 python -m pytest tests/test_tc_bwd.py tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -2
bash tools/gpu/ab_multi.sh kwprev
for d in 4 16 32; do echo "GLA_KW_DBG=$d: $(GLA_KW_DBG=$d timeout 200 python tools/kbench.py 1p3b 2>&1 | grep -E 'bwd_dq|bwd_dk' | tr -s ' ' | tr '\n' ';')"; done
