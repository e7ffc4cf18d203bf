mkdir -p gpurun_out
for kern in k_fwd_prep k_bwd_reduce_tma; do
  ncu --set full --clock-control none --import-source on -k "regex:$kern" -s 1 -c 1 -o gpurun_out/exact_$kern -f python tools/mixed_step.py > gpurun_out/exact_$kern.log 2>&1
  ncu -i gpurun_out/exact_$kern.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/exact_${kern}_src.csv 2>/dev/null
  ncu -i gpurun_out/exact_$kern.ncu-rep --page details --csv > gpurun_out/exact_${kern}_details.csv 2>/dev/null
  tail -2 gpurun_out/exact_$kern.log
done
