timeout 600 python -m pytest tests/test_tc_bwd.py -m gpu -q -k "deterministic" 2>&1 | tail -3
