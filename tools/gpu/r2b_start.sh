# Session-3 start: full GPU suite, smoke, bench line, per-kernel timing, mixed-gate step.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -6 | tee gpurun_out/r2b_gputests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 600 python bench.py > gpurun_out/r2b_bench.json 2> gpurun_out/r2b_bench.err; tail -c 800 gpurun_out/r2b_bench.json
timeout 300 python tools/kbench.py 1p3b 2>&1 | tail -16
timeout 300 python tools/mixed_step.py 2>&1 | tail -8
