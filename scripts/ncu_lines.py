"""Aggregate an `ncu --page source --print-source cuda,sass --csv` dump per
CUDA source line: warp instructions executed and stall samples."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
f = None
agg = {}
hdr = None
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8 or r[0] == "" or r[0] == "Function Name":
        continue
    try:
        inst = float(r[7]); samp = float(r[4])
    except ValueError:
        continue
    key = (f, r[0])
    a = agg.setdefault(key, [0.0, 0.0, r[1][:90]])
    a[0] += inst; a[1] += samp
ti = sum(a[0] for a in agg.values()) or 1
ts = sum(a[1] for a in agg.values()) or 1
for (f, ln), (i, s, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{f}:{ln:>4} inst {100*i/ti:5.1f}% stall {100*s/ts:5.1f}%  {src}")
