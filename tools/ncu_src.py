"""Summarise an `ncu --page source --csv --print-source cuda,sass` dump: top source lines by stall samples."""
import csv
import sys

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
rows = list(csv.reader(open(path)))
cur_file = None
agg = []
hdr = None
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and r and r[0].isdigit():
        d = dict(zip(hdr, r))
        try:
            s = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
        except ValueError:
            s = 0
        stalls = {k: int(v) for k, v in d.items() if k.startswith("stall_") and "Not Issued" not in k and v.isdigit() and int(v) > 0}
        agg.append((s, cur_file, r[0], r[1][:90], sorted(stalls.items(), key=lambda x: -x[1])[:3]))
tot = sum(a[0] for a in agg)
agg.sort(key=lambda x: -x[0])
print("total samples", tot)
for s, f, ln, src, st in agg[:top]:
    print(f"{100*s/max(tot,1):5.1f}% {f}:{ln} {src} {st}")
