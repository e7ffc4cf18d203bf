# kwalk timing experiments (results wrong when GLA_KW_DBG is set): 4 = epilogue only drains, 8 = no output MMAs
for d in 0 4 8 12; do echo "== GLA_KW_DBG=$d"; GLA_KW_DBG=$d timeout 120 python tools/kbench.py 1p3b 2>&1 | grep 'bwd_d[qk]'; done
