"""Dump frame 0's merged C3 mesh (+ rig) to gpurun_out/ for offline raster
statistics (per-(camera, triangle) bbox / candidate / inside counts).
Run on the GPU box: python scripts/dump_c3_mesh.py [workload]."""

import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1903_11785_b200 import synthetic as S, workloads  # noqa: E402
from paper_1903_11785_b200.pipeline import run_frame  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
wl = workloads.get(name)
masks, frames = S.render_scene_device(wl.rig, wl.objects(0), shade=True)
torch.cuda.synchronize()
m = masks.cpu().numpy()
sils = [m[i].astype(bool) for i in range(m.shape[0])]
fr = {c.id: frames[i].cpu().numpy() for i, c in enumerate(wl.rig)}
b = run_frame(wl.cfg, wl.rig, fr, sils=sils)
mm = b.merged_mesh
os.makedirs("gpurun_out", exist_ok=True)
cams = list(wl.rig)
np.savez_compressed(f"gpurun_out/{name}_mesh.npz", verts=mm.vertices, tris=mm.triangles,
                    R=np.stack([c.rotation for c in cams]), t=np.stack([c.translation for c in cams]),
                    K=np.array([[c.fx, c.fy, c.cx, c.cy, c.skew, c.image_width, c.image_height] for c in cams]))
print("dumped", mm.vertices.shape, mm.triangles.shape)
