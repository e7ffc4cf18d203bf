"""Top source lines by warp-stall samples from an `ncu --page source --csv --print-source cuda,sass` export
(CUDA-source rows only), with the dominant stall reasons.  python tools/ncu_src_top.py file.csv [n]"""
import csv
import sys

n_top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
rows = []
path = None
hdr = None
with open(sys.argv[1]) as f:
    for r in csv.reader(f):
        if not r:
            continue
        if r[0] == "File Path":
            path = r[1].split("/")[-1]
            hdr = None
            continue
        if r[0] == "Function Name":
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or not r[0].isdigit():
            continue
        d = dict(zip(hdr, r))
        try:
            samp = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
        except ValueError:
            continue
        stalls = {k: int(v) for k, v in d.items() if k.startswith("stall_") and "Not Issued" not in k and v.isdigit()}
        rows.append((samp, path, r[0], r[1][:90], sorted(stalls.items(), key=lambda x: -x[1])[:3]))
tot = sum(x[0] for x in rows)
print(f"total samples {tot}")
for samp, path, ln, src, st in sorted(rows, key=lambda x: -x[0])[:n_top]:
    print(f"{100 * samp / max(tot, 1):5.1f}% {path}:{ln} {src.strip()} | " + ", ".join(f"{k[6:]}={v}" for k, v in st))
