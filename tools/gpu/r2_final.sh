# Round-2 final evidence on one B200: full GPU test suite, smoke, sanitizers, bench line, launch list, sweeps.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -4 | tee gpurun_out/r2_gputests_final.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
rm -f gpurun_out/sanitize_final.txt
for tool in memcheck racecheck synccheck; do
  echo "== $tool" >> gpurun_out/sanitize_final.txt
  timeout 1500 compute-sanitizer --tool $tool --print-limit 10 python tools/sanitize_small.py >> gpurun_out/sanitize_final.txt 2>&1
  echo "rc=$?" >> gpurun_out/sanitize_final.txt
done
grep -E '^==|SUMMARY|rc=|sanitize_small' gpurun_out/sanitize_final.txt
timeout 600 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; tail -c 600 gpurun_out/bench_final.json
timeout 900 python tools/sweep.py > gpurun_out/r2_sweep_final.md 2> gpurun_out/r2_sweep_final.err; cat gpurun_out/r2_sweep_final.md
timeout 900 python tools/chunk_sweep.py --out gpurun_out/r2_chunk_sweep.md > /dev/null 2>&1; cat gpurun_out/r2_chunk_sweep.md
