"""Print (id, kernel, µs) from an ncu --metrics gpu__time_duration.sum csv."""
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/launches_r.csv"))
        if len(r) > 10]
h = rows[0]
iK, iM, iV, iI = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
for r in rows[1:]:
    if r[iM] == "gpu__time_duration.sum":
        print(r[iI], r[iK].split("(")[0][:40], round(float(r[iV]) / 1000, 1))
