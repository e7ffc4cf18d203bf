# Full round evidence on one B200: GPU tests, smoke, bench line, ncu launch list, one ncu --set full capture of
# every kernel of a step (summarised to profiles/-ready JSON by tools/ncu_summary.py).
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -4
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -c 3000 gpurun_out/bench.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_(fwd_prep|fwd_state|bwd_dp|bwd_dq3|bwd_dkv3|bwd_reduce_tma|bwd_gate)" -s 7 -c 7 -o gpurun_out/step_full -f python tools/kbench.py > gpurun_out/ncu_full.log 2>&1
python tools/ncu_summary.py gpurun_out/step_full.ncu-rep gpurun_out/ncu_summary.json; cat gpurun_out/ncu_summary.json | head -80
