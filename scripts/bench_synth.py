"""f4 measurement: the reference's Sphere/Box scene generator on the GPU,
16 cameras 1920x1080 (C3 rig), 12 spheres + 12 boxes: device time of
fvv_synth_render (silhouette + frame) per camera and the public-API time of
scene_silhouettes + scene_frames (host arrays out)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1903_11785_b200 import synthetic as S

rig = S.ring_rig(16, (0, 0, 1000), 15000, 4000, 1920, 1080, 1600)
rng = np.random.default_rng(0)
objs = []
for i in range(12):
    x, y = rng.uniform(-8000, 8000), rng.uniform(-3800, 3800)
    objs.append(S.Sphere(center=[x, y, 900], radius=rng.uniform(200, 500)))
    objs.append(S.Box(lo=[x + 600, y, 0], hi=[x + 900, y + 300, 1800]))
scene = S.SyntheticScene(rig=rig, objects=objs)
cams = list(rig)
for _ in range(2):
    S._synth_device(cams[0], objs, scene.light_dir, True, True)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for cam in cams:
    S._synth_device(cam, objs, scene.light_dir, True, True)
b.record(); torch.cuda.synchronize()
dev_ms = a.elapsed_time(b)
t = time.perf_counter()
sils = S.scene_silhouettes(scene)
frames = S.scene_frames(scene)
api_s = time.perf_counter() - t
print(f"16 x 1080p, {len(objs)} objects: device {dev_ms:.2f} ms for all cameras "
      f"(silhouette + frame); public API {api_s * 1e3:.1f} ms "
      f"(fg fraction {np.mean([s.mean() for s in sils]):.3f})")
