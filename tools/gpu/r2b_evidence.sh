# Session-3 evidence on one B200: GPU suite, smoke, ncu --set full of every kernel of a 1.3B step (summary ->
# profiles/ncu_summary_latest.json, read by bench.py's roofline), bench line, ncu launch list, 2-rank and sp32k lines,
# sweep of every config (incl. guard cliff and cold-state decode).
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -4 | tee gpurun_out/r2b_gputests_final.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_fwd_prep|k_fwd_state|k_bwd_dp|k_bwd_kwalk|k_bwd_dkv3|k_bwd_reduce_tma|k_bwd_gate" -s 8 -c 8 -o gpurun_out/step_full -f python tools/kbench.py > gpurun_out/ncu_full.log 2>&1
python tools/ncu_summary.py gpurun_out/step_full.ncu-rep gpurun_out/ncu_summary.json
cp gpurun_out/ncu_summary.json profiles/ncu_summary_latest.json
timeout 600 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; tail -c 1500 gpurun_out/bench_final.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_final.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 600 python bench.py --gpus 2 --steps 5 --warmup 3 --no-e2e > gpurun_out/bench_g2.json 2> gpurun_out/bench_g2.err; tail -c 600 gpurun_out/bench_g2.json
timeout 900 python bench.py --config sp32k --steps 5 --warmup 3 > gpurun_out/bench_sp1.json 2>&1; tail -c 600 gpurun_out/bench_sp1.json
timeout 1200 python tools/sweep.py > gpurun_out/sweep_final.md 2> gpurun_out/sweep_final.err; cat gpurun_out/sweep_final.md
python - <<'PY'
import json
d = json.load(open("gpurun_out/ncu_summary.json"))
for k, v in d.items():
    print(f"{k[:60]:60s} {v.get('duration', 0)*1e6:8.1f} us  dram {v.get('traffic_bytes', 0)/1e6:8.1f} MB  tensor {v.get('tensor_pipe_pct', 0):5.1f}%")
PY
