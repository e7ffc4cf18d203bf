for e in "GLA_DV_LAST=1" "X=1"; do echo "== $e"; for r in 1 2; do env $e timeout 120 python tools/kbench.py 1p3b 2>&1 | grep 'step'; done; done
timeout 600 python -m pytest tests/test_tc_bwd.py -m gpu -x -q 2>&1 | tail -2
