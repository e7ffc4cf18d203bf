mkdir -p gpurun_out
for kern in k_out_bwd k_prep_bwd "k_prep<" "k_out<"; do
  tag=$(echo $kern | tr -d '<')
  timeout 600 ncu --set full --clock-control none --import-source on -k "regex:$kern" -s 1 -c 1 -o gpurun_out/nl_$tag -f python tools/layer_bench.py > gpurun_out/nl_$tag.log 2>&1
  ncu -i gpurun_out/nl_$tag.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/nl_${tag}_src.csv 2>/dev/null
  ncu -i gpurun_out/nl_$tag.ncu-rep --page details --csv > gpurun_out/nl_${tag}_details.csv 2>/dev/null
  echo "=== $kern"; python tools/ncu_src_top.py gpurun_out/nl_${tag}_src.csv 8
  python - "$tag" <<'PY'
import csv, sys
rows = list(csv.reader(open(f"gpurun_out/nl_{sys.argv[1]}_details.csv")))
hdr = rows[0]
for r in rows[1:]:
    d = dict(zip(hdr, r))
    n = d.get("Metric Name", "")
    if n in ("Duration", "DRAM Throughput", "Achieved Occupancy", "Registers Per Thread", "Issue Slots Busy"):
        print("   ", n, d["Metric Unit"], d["Metric Value"])
PY
done
