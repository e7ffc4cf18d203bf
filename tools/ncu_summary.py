"""Summarise an ncu --set full report: per kernel duration, DRAM bytes, pipe utilisation, occupancy.
python tools/ncu_summary.py report.ncu-rep out.json"""
import csv
import io
import json
import subprocess
import sys

rep, out = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
want = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active": "tensor_pipe_pct",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active": "xu_pipe_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "launch__registers_per_thread": "registers",
    "lts__t_bytes.sum": "l2_bytes",
}
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "usecond": 1e-6, "us": 1e-6, "ns": 1e-9, "ms": 1e-3,
         "msecond": 1e-3, "nsecond": 1e-9}
res = {}
for r in rows[2:]:
    d = dict(zip(hdr, r))
    name = d.get("Kernel Name", "?").split("(")[0].replace("void ", "")
    entry = {}
    for k, short in want.items():
        if k in d and d[k] not in ("", "n/a"):
            u = units[hdr.index(k)]
            v = float(d[k].replace(",", ""))
            entry[short] = v * scale.get(u, 1) if u in scale else v
    entry["traffic_bytes"] = entry.get("dram_read", 0) + entry.get("dram_write", 0)
    res.setdefault(name, []).append(entry)
summary = {}
for name, es in res.items():
    avg = {k: sum(e.get(k, 0) for e in es) / len(es) for k in es[0]}
    avg["captures"] = len(es)
    summary[name] = avg
json.dump(summary, open(out, "w"), indent=1)
for n, a in summary.items():
    print(f"{n:60s} {a.get('duration', 0) * 1e6:8.1f} us  DRAM {a['traffic_bytes'] / 1e6:8.1f} MB  "
          f"tensor {a.get('tensor_pipe_pct', 0):5.1f}%  dram {a.get('dram_pct', 0):5.1f}%  issue {a.get('issue_active_pct', 0):5.1f}%")
