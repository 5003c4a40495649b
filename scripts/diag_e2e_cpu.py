"""e2e (run_sequence, C3, 4 lanes) wall vs host CPU time per frame: is the
end-to-end rate bound by the caller's Python thread?"""
import gc
import sys as _sys
if len(_sys.argv) > 1:
    _sys.setswitchinterval(float(_sys.argv[1]))
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1903_11785_b200 import synthetic as S, workloads
from paper_1903_11785_b200.pipeline import run_sequence

wl = workloads.get("C3")
cams = list(wl.rig)
host = []
for f in range(4):
    masks, frames = S.render_scene_device(wl.rig, wl.objects(f), shade=True)
    fr = {c.id: t for c, t in zip(cams, frames.cpu().pin_memory())}
    host.append((masks.cpu().pin_memory(), fr))


def run(n, consume=True):
    fr = [host[i % 4][1] for i in range(n)]
    ms = [host[i % 4][0] for i in range(n)]
    busy = 0.0
    for b, img in run_sequence(wl.cfg, wl.rig, fr, ms, wl.virtual, lanes=4):
        if consume:
            b.merged_mesh.vertices.shape, img.color.shape


run(12)
torch.cuda.synchronize()
gc.collect()
gc.disable()
n = 80
t0, c0, m0 = time.perf_counter(), os.times(), time.thread_time()
run(n)
torch.cuda.synchronize()
t1, c1, m1 = time.perf_counter(), os.times(), time.thread_time()
wall = (t1 - t0) / n * 1e3
cpu = ((c1.user - c0.user) + (c1.system - c0.system)) / n * 1e3
print(f"wall {wall:.3f} ms/frame ({1e3 / wall:.0f} fps); process CPU {cpu:.3f} ms/frame; "
      f"caller thread CPU {(m1 - m0) / n * 1e3:.3f} ms/frame")
