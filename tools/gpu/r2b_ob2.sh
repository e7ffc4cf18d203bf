# fwd_state with two output accumulators (OB2): forward parity, A/B against the ordered single accumulator, phase traces.
timeout 900 python -m pytest tests/test_tc_fwd.py tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -2
bash tools/gpu/ab_multi.sh ob1
timeout 200 python tools/phase_timing.py 1p3b 2>&1 | tail -16
cp variants/libgla_timing_ob1.so paper_2312_06635_b200/libgla_timing.so
timeout 200 python tools/phase_timing.py 1p3b 2>&1 | tail -16
