mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k "regex:k_bwd_reduce_tma|k_fwd_prep|k_bwd_dp" -s 6 -c 3 -o gpurun_out/bw3 -f python tools/kbench.py 1p3b > gpurun_out/bw3.log 2>&1
ncu -i gpurun_out/bw3.ncu-rep --page details --csv > gpurun_out/bw3_details.csv 2>/dev/null
ncu -i gpurun_out/bw3.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/bw3_src.csv 2>/dev/null
tail -2 gpurun_out/bw3.log
