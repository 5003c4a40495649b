"""Which transfer bounds run_sequence's end-to-end rate? C3, 4 lanes: pinned
host silhouettes (as bench.py) vs. silhouettes already on the device."""
import gc
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1903_11785_b200 import synthetic as S, workloads
from paper_1903_11785_b200.pipeline import run_sequence

wl = workloads.get("C3")
cams = list(wl.rig)
host, dev = [], []
for f in range(4):
    masks, frames = S.render_scene_device(wl.rig, wl.objects(f), shade=True)
    fr = {c.id: t for c, t in zip(cams, frames.cpu().pin_memory())}
    host.append((masks.cpu().pin_memory(), fr))
    dev.append((masks.clone(), fr))


def run(src, n, lanes):
    fr = [src[i % 4][1] for i in range(n)]
    ms = [src[i % 4][0] for i in range(n)]
    for b, img in run_sequence(wl.cfg, wl.rig, fr, ms, wl.virtual, lanes=lanes):
        b.merged_mesh.vertices.shape, img.color.shape


for lanes in (4, 6):
    for name, src in (("host sils", host), ("device sils", dev)):
        run(src, 12, lanes)
        torch.cuda.synchronize()
        gc.collect()
        gc.disable()
        t = time.perf_counter()
        run(src, 80, lanes)
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t) / 80 * 1e3
        gc.enable()
        print(f"lanes {lanes} {name}: {dt:.3f} ms/frame ({1e3 / dt:.1f} fps)")
