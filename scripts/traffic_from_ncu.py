"""profiles/traffic.json from an `ncu --set full` report of one C3 frame's
carve and raster kernels: DRAM bytes (dram__bytes_read.sum +
dram__bytes_write.sum) per kernel launch, grouped as bench.py reads them.

  python scripts/traffic_from_ncu.py gpurun_out/r1_v8_full.ncu-rep
"""
import csv
import io
import json
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                      "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"],
                     capture_output=True, text=True, check=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, units = rows[0], rows[1]
iK, iR, iW, iT = (h.index(n) for n in ("Kernel Name", "dram__bytes_read.sum",
                                        "dram__bytes_write.sum", "gpu__time_duration.sum"))
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
launches = []
for r in rows[2:]:
    name = r[iK].split("(")[0]
    b = float(r[iR]) * scale[units[iR]] + float(r[iW]) * scale[units[iW]]
    launches.append((name, b, float(r[iT])))
carve = [b for n, b, _ in launches if n == "carve_kernel"][:2]  # B-1, B-3 of the first frame
d1 = []  # first D-1 launch group: prep .. big (16 cameras)
for n, b, _ in launches:
    if n == "raster_prep_kernel" and d1:
        break
    if n.startswith("raster_"):
        d1.append((n, b))
src = f"{rep} (ncu --set full, first C3 frame; dram__bytes_read.sum + dram__bytes_write.sum)"
out = {
    "carve_kernel": {"bytes_per_launch": int(sum(carve) / len(carve)),
                     "launches": [int(b) for b in carve], "source": src},
    "depth_images": {"bytes": int(sum(b for _, b in d1)),
                     "kernels": {n: int(b) for n, b in d1}, "source": src},
}
json.dump(out, open("profiles/traffic.json", "w"), indent=1)
print(json.dumps(out, indent=1))
