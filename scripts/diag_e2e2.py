"""Replicates bench.py's e2e leg and prints per-frame intervals."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1903_11785_b200 import workloads, synthetic as S
from paper_1903_11785_b200.pipeline import run_sequence
wl = workloads.get("C3"); cams = list(wl.rig)
host = []
for f in range(4):
    masks, frames = S.render_scene_device(wl.rig, wl.objects(f), shade=True)
    host.append((masks.cpu().pin_memory(), {c.id: t for c, t in zip(cams, frames.cpu().pin_memory())}))
def run(n, label):
    fr = [host[i % 4][1] for i in range(n)]; ms = [host[i % 4][0] for i in range(n)]
    torch.cuda.synchronize(); t0 = time.perf_counter(); ts = []
    for b, img in run_sequence(wl.cfg, wl.rig, fr, ms, wl.virtual):
        b.merged_mesh.object_ids; ts.append(time.perf_counter())
    torch.cuda.synchronize(); t1 = time.perf_counter()
    d = np.diff([t0] + ts) * 1e3
    print(f"{label}: {(t1 - t0) / n * 1e3:.2f} ms/frame; intervals: " + " ".join(f"{x:.1f}" for x in d))
run(3, "warm")
for r in range(4):
    run(30, f"timed{r}")
