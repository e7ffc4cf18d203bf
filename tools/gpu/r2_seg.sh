timeout 900 python -m pytest tests/test_tc_bwd.py tests/test_tc_fwd.py -m gpu -q -x 2>&1 | tail -2
for c in t4k t8k long16k 340m 1p3b; do echo "$c $(timeout 200 python tools/kbench.py $c 2>&1 | grep 'step (wall')"; done
