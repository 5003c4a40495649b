"""Per-source-line instruction / stall totals of one kernel launch in an ncu
report (--print-source cuda,sass): python scripts/ncu_lines.py REP SKIP [N]"""
import csv
import io
import subprocess
import sys

rep, skip = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                      "cuda,sass", "--launch-skip", skip, "--launch-count", "1"],
                     capture_output=True, text=True).stdout
fname, rows, hdr = None, [], None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr and r[0] not in ("", "Function Name"):
        try:
            rows.append((fname, r[0], r[1], int(r[hdr.index("Warp Stall Sampling (All Samples)")]),
                         int(r[hdr.index("Instructions Executed")])))
        except ValueError:
            pass
ts = sum(x[3] for x in rows) or 1
ti = sum(x[4] for x in rows) or 1
print(f"total stall samples {ts}, warp instructions {ti}")
for f, ln, src, s, n in sorted(rows, key=lambda x: -x[3])[:top]:
    print(f"{s / ts * 100:5.1f}% stall {n / ti * 100:5.1f}% inst  {f}:{ln}  {src.strip()[:70]}")
