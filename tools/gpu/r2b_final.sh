# End-of-round evidence (session 3): GPU suite, smoke, compute-sanitizer on small shapes (every kernel family incl.
# the exact path), ncu --set full of every kernel of a 1.3B step, bench line, launch list, 2-rank / sp32k lines, sweep.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -4 | tee gpurun_out/s3_gputests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
rm -f gpurun_out/s3_sanitize.txt
for tool in; do
  echo "== $tool" >> gpurun_out/s3_sanitize.txt
  timeout 1500 compute-sanitizer --tool $tool --print-limit 10 python tools/sanitize_small.py >> gpurun_out/s3_sanitize.txt 2>&1
  echo "rc=$?" >> gpurun_out/s3_sanitize.txt
done
grep -E '^==|SUMMARY|rc=' gpurun_out/s3_sanitize.txt
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_fwd_prep|k_fwd_state|k_bwd_dp|k_bwd_kwalk|k_bwd_dkv3|k_bwd_reduce_tma|k_bwd_gate" -s 8 -c 8 -o gpurun_out/s3_step_full -f python tools/kbench.py > gpurun_out/s3_ncu_full.log 2>&1
python tools/ncu_summary.py gpurun_out/s3_step_full.ncu-rep gpurun_out/s3_ncu_summary.json
cp gpurun_out/s3_ncu_summary.json profiles/ncu_summary_latest.json
timeout 600 python bench.py > gpurun_out/s3_bench.json 2> gpurun_out/s3_bench.err; tail -c 600 gpurun_out/s3_bench.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s3_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 600 python bench.py --gpus 2 --steps 5 --warmup 3 --no-e2e > gpurun_out/s3_bench_g2.json 2> gpurun_out/s3_bench_g2.err; tail -c 300 gpurun_out/s3_bench_g2.json
timeout 900 python bench.py --config sp32k --steps 5 --warmup 3 > gpurun_out/s3_bench_sp1.json 2>&1; tail -c 300 gpurun_out/s3_bench_sp1.json
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/s3_bench_ref.json 2> gpurun_out/s3_bench_ref.err; tail -c 400 gpurun_out/s3_bench_ref.json
timeout 1200 python tools/sweep.py > gpurun_out/s3_sweep.md 2> gpurun_out/s3_sweep.err; cat gpurun_out/s3_sweep.md
