mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:k_out_bwd" -s 1 -c 1 -o gpurun_out/n_outb -f python tools/layer_bench.py > gpurun_out/n_outb.log 2>&1
ncu -i gpurun_out/n_outb.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/n_outb_src.csv 2>/dev/null
ncu -i gpurun_out/n_outb.ncu-rep --page details --csv > gpurun_out/n_outb_details.csv 2>/dev/null
python tools/ncu_src_top.py gpurun_out/n_outb_src.csv 16
