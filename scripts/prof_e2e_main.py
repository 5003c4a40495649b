"""cProfile of the caller's thread in run_sequence (4 lanes, C3), bench-like consumer."""
import cProfile, pstats, sys, os, time, gc
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1903_11785_b200 import workloads, synthetic as S
from paper_1903_11785_b200.pipeline import run_sequence
wl = workloads.get("C3"); cams = list(wl.rig)
host = []
for f in range(4):
    masks, frames = S.render_scene_device(wl.rig, wl.objects(f), shade=True)
    host.append((masks.cpu().pin_memory(), {c.id: t for c, t in zip(cams, frames.cpu().pin_memory())}))
def d2h(bundle, img):
    m = bundle.merged_mesh
    return m.vertices.shape[0] + m.triangles.shape[0] + img.color.shape[0]  # as bench.py
def run(n):
    fr = [host[i % 4][1] for i in range(n)]; ms = [host[i % 4][0] for i in range(n)]
    tot = 0
    for b, img in run_sequence(wl.cfg, wl.rig, fr, ms, wl.virtual):
        tot += d2h(b, img)
    return tot
run(12); torch.cuda.synchronize(); gc.collect(); gc.disable()
t = time.perf_counter(); run(60); torch.cuda.synchronize(); print("e2e ms/frame", (time.perf_counter() - t) / 60 * 1e3)
pr = cProfile.Profile(); pr.enable(); run(60); torch.cuda.synchronize(); pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(30)
