"""bench.py's e2e leg repeated: per-frame intervals, GC events, to find stalls."""
import sys, os, time, gc
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1903_11785_b200 import workloads, synthetic as S
from paper_1903_11785_b200.pipeline import run_sequence
from paper_1903_11785_b200.executor import executor_for
wl = workloads.get("C3"); cams = list(wl.rig)
inputs = [S.render_scene_device(wl.rig, wl.objects(f), shade=True) for f in range(4)]
ex = executor_for(wl.cfg, wl.rig)
for i in range(13):  # the device leg
    m, fr = inputs[i % 4]
    ex.run(m, wl.virtual, fr.reshape(-1), np.arange(16, dtype=np.int64) * (1080 * 1920 * 3))
torch.cuda.synchronize()
host = [(m.cpu().pin_memory(), {c.id: t for c, t in zip(cams, f.cpu().pin_memory())}) for m, f in inputs]
EV = []
gc.callbacks.append(lambda ph, info: EV.append((time.perf_counter(), ph, info["generation"])))
def run(n, lanes=2):
    fr = [host[i % 4][1] for i in range(n)]; ms = [host[i % 4][0] for i in range(n)]
    EV.clear(); torch.cuda.synchronize(); t0 = time.perf_counter(); ts = []
    for b, img in run_sequence(wl.cfg, wl.rig, fr, ms, wl.virtual, lanes=lanes):
        b.merged_mesh.triangles; ts.append(time.perf_counter())
    torch.cuda.synchronize(); t1 = time.perf_counter()
    d = np.diff([t0] + ts) * 1e3
    gcs = [f"{(t - t0) * 1e3:.1f}:{ph[0]}{g}" for t, ph, g in EV]
    return (t1 - t0) / n * 1e3, d, gcs
for lanes in (1, 2, 3, 4):
    run(12, lanes)
    for r in range(3):
        ms, d, gcs = run(30, lanes)
        print(f"lanes {lanes} rep {r}: {ms:.2f} ms/frame ({1e3 / ms:.0f} fps)  first intervals " + " ".join(f"{x:.1f}" for x in d[:6]))
