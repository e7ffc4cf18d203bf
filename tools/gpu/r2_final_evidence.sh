# Round-2 evidence: ncu --set full of every kernel of one 1.3B step (summary -> profiles/ncu_summary_latest.json
# so bench.py's roofline carries the measured DRAM bytes), the bench line, the ncu launch list of the bench command.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_fwd_prep|k_fwd_state|k_bwd_dp|k_bwd_kwalk|k_bwd_dkv3|k_bwd_reduce_tma|k_bwd_gate" -s 8 -c 8 -o gpurun_out/step_full -f python tools/kbench.py > gpurun_out/ncu_full.log 2>&1
python tools/ncu_summary.py gpurun_out/step_full.ncu-rep gpurun_out/ncu_summary.json
cp gpurun_out/ncu_summary.json profiles/ncu_summary_latest.json
timeout 600 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; tail -c 1500 gpurun_out/bench_final.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_final.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
python - <<'PY'
import json
d = json.load(open("gpurun_out/ncu_summary.json"))
for k, v in d.items():
    print(f"{k[:60]:60s} {v.get('duration', 0)*1e6:8.1f} us  dram {v.get('traffic_bytes', 0)/1e6:8.1f} MB  tensor {v.get('tensor_pipe_pct', 0):5.1f}%")
PY
