"""Host-side profile of the device frame loop (cProfile), C3 workload."""
import cProfile, pstats, sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1903_11785_b200 import workloads, synthetic as S
from paper_1903_11785_b200._device import DeviceSilhouettes
from paper_1903_11785_b200.pipeline import reconstruct
from paper_1903_11785_b200.render import render_device
wl = workloads.get("C3"); cams = list(wl.rig)
masks, frames = S.render_scene_device(wl.rig, wl.objects(0))
fb = frames.reshape(-1); foff = np.arange(16, dtype=np.int64) * (1080 * 1920 * 3)
def step():
    d = DeviceSilhouettes(wl.rig, masks)
    r = reconstruct(wl.cfg, wl.rig, d)
    render_device(r.batch.verts, r.batch.tris, int(r.batch.tris.shape[0]), cams, None, r.vis_bits,
                  int(r.vis_bits.shape[1]), wl.virtual, nt_dev=r.batch.num_triangles_dev,
                  frame_buf=(fb, foff))
for _ in range(3): step()
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(10): step()
torch.cuda.synchronize(); print("ms/step", (time.perf_counter() - t) * 100)
pr = cProfile.Profile(); pr.enable()
for _ in range(10): step()
torch.cuda.synchronize(); pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
