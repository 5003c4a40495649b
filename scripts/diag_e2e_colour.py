import sys, os, time, gc
sys.path.insert(0, "/root/repo")
import numpy as np, torch
from paper_1903_11785_b200 import workloads, synthetic as S
from paper_1903_11785_b200.pipeline import run_sequence
wl = workloads.get("C3"); cams = list(wl.rig)
host = []
for f in range(4):
    masks, frames = S.render_scene_device(wl.rig, wl.objects(f), shade=True)
    host.append((masks.cpu().pin_memory(), {c.id: t for c, t in zip(cams, frames.cpu().pin_memory())}))
def run(n, virt, lanes=4):
    fr = [host[i % 4][1] for i in range(n)]; ms = [host[i % 4][0] for i in range(n)]
    for b, img in run_sequence(wl.cfg, wl.rig, fr, ms, virt, lanes=lanes):
        b.merged_mesh.triangles
gc.disable()
for virt, name in ((wl.virtual, "with colour"), (None, "no colour")):
    run(12, virt); torch.cuda.synchronize()
    t = time.perf_counter(); run(80, virt); torch.cuda.synchronize()
    print(name, f"{(time.perf_counter() - t) / 80 * 1e3:.3f} ms/frame")
