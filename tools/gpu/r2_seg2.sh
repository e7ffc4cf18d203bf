timeout 1200 python -m pytest tests/test_tc_bwd.py tests/test_tc_fwd.py tests/test_parallel.py -m gpu -q -x 2>&1 | tail -2
for c in t8k long16k long32k; do echo "$c $(timeout 200 python tools/kbench.py $c 2>&1 | grep 'step (wall')"; done
timeout 300 python tools/kbench.py long16k 2>&1 | grep summary
