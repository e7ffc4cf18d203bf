# usage: bash tools/gpu/ncu_kernel.sh <kernel regex> <tag>   -- one --set full capture of the kernel in kbench
set -e
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k "regex:$1" -s ${3:-3} -c 1 -o gpurun_out/$2 -f python tools/kbench.py ${4:-1p3b} > gpurun_out/$2.log 2>&1 || true
ncu -i gpurun_out/$2.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/$2_src.csv 2>/dev/null || true
ncu -i gpurun_out/$2.ncu-rep --page details --csv > gpurun_out/$2_details.csv 2>/dev/null || true
tail -3 gpurun_out/$2.log
