# Timing experiments on the K-tiled walks (results wrong when set): 4 = epilogue only drains, 8 = no output MMAs.
for d in 0 4 16 32 48; do echo "GLA_KW_DBG=$d: $(GLA_KW_DBG=$d timeout 200 python tools/kbench.py 1p3b 2>&1 | grep -E 'bwd_dq|bwd_dk' | tr -s ' ' | tr '\n' ';')"; done
