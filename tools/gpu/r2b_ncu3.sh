# ncu --set full (with source) of the dv walk, the forward prep and the backward dP kernel at 1.3B shapes.
mkdir -p gpurun_out
for kern in "k_bwd_dkv3" "k_fwd_prep" "k_bwd_dp" "k_bwd_reduce_tma"; do
  timeout 600 ncu --set full --clock-control none --import-source on -k "regex:$kern" -s 2 -c 1 -o gpurun_out/n3_$kern -f python tools/kbench.py 1p3b > gpurun_out/n3_$kern.log 2>&1
  ncu -i gpurun_out/n3_$kern.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/n3_${kern}_src.csv 2>/dev/null
  ncu -i gpurun_out/n3_$kern.ncu-rep --page details --csv > gpurun_out/n3_${kern}_details.csv 2>/dev/null
  python tools/ncu_src_top.py gpurun_out/n3_${kern}_src.csv 14 2>&1 | head -16
done
