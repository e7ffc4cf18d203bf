# Per-kernel timing only (no tests): 1.3B and 340M steps.
timeout 300 python tools/kbench.py 1p3b 2>&1 | tail -11
timeout 300 python tools/kbench.py 340m 2>&1 | tail -11
