timeout 1200 python tools/dlog_err.py 2>&1 | tail -8 | tee gpurun_out/dlog_err.md
