mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k "regex:k_bwd_dq|k_fwd_state" -c 2 -o gpurun_out/simt2 -f python tools/simt_breakdown.py > gpurun_out/simt2.log 2>&1
ncu -i gpurun_out/simt2.ncu-rep --page details --csv > gpurun_out/simt2_details.csv 2>/dev/null
ncu -i gpurun_out/simt2.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/simt2_src.csv 2>/dev/null
tail -2 gpurun_out/simt2.log
