# kwalk A/B (GLA_KW_DBG=16: one output issuer)
for d in 0 16; do echo "== GLA_KW_DBG=$d"; GLA_KW_DBG=$d timeout 120 python tools/kbench.py 1p3b 2>&1 | grep 'bwd_d[qk]\|step'; done
GLA_KW_DBG=16 timeout 600 python -m pytest tests/test_tc_bwd.py -m gpu -x -q 2>&1 | tail -2
