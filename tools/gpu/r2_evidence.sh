# Round 2 evidence on one B200: GPU tests, smoke, default bench line, ncu launch list, multi-rank modes.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -8 | tee gpurun_out/r2_gputests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 600 python bench.py > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err; tail -c 4000 gpurun_out/r2_bench.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 600 python bench.py --gpus 2 --steps 5 --warmup 3 --no-e2e > gpurun_out/r2_bench_g2.json 2> gpurun_out/r2_bench_g2.err; tail -c 1500 gpurun_out/r2_bench_g2.json
timeout 900 python bench.py --config sp32k --steps 5 --warmup 3 > gpurun_out/r2_sp1.json 2>&1; tail -c 1500 gpurun_out/r2_sp1.json
