for s in "" 2 4; do echo "== 340m GLA_SEGMENTS=$s"; GLA_SEGMENTS=$s timeout 200 python tools/kbench.py 340m 2>&1 | tail -14; done
