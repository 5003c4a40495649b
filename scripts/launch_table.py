"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list:
per-kernel time per frame and share (harness input generation excluded)."""
import collections
import csv
import sys

path = sys.argv[1]
frames = float(sys.argv[2]) if len(sys.argv) > 2 else 3.0
rows = list(csv.reader(open(path)))
hdr = None
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        name = d["Kernel Name"].split("(")[0].replace("void ", "")
        if "render_parts" in name:
            continue
        v = float(d["Metric Value"]) * {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0,
                                         "ms": 1e3, "msecond": 1e3}[d["Metric Unit"]]
        agg[name][0] += 1
        agg[name][1] += v
tot = sum(v[1] for v in agg.values())
print(f"{'kernel':58s} {'us/frame':>9s} {'share':>6s} launches")
for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k[:58]:58s} {v[1] / frames:9.1f} {100 * v[1] / tot:5.1f}% {v[0]}")
print(f"{'total':58s} {tot / frames:9.1f}")
