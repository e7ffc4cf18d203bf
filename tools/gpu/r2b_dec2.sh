for n in 1 4 8 16 64; do echo "GLA_STEP_NARROW=$n"; GLA_STEP_NARROW=$n SWEEP_DECODE_ONLY=1 timeout 600 python tools/sweep.py 2>&1 | tail -4; done
