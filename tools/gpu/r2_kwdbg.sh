# kwalk timing experiments (results wrong when GLA_KW_DBG is set)
for d in 0 16 8; do for c in 1p3b 340m; do echo "== GLA_KW_DBG=$d $c"; GLA_KW_DBG=$d timeout 120 python tools/kbench.py $c 2>&1 | grep 'bwd_d[qk]\|step'; done; done
