"""Quick timing probe: C3-scale coarse carve on the GPU vs the oracle."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle as O
from paper_1903_11785_b200 import synthetic as S
from paper_1903_11785_b200.hull import carve, carve_grids
from paper_1903_11785_b200._device import DeviceSilhouettes
from paper_1903_11785_b200.voxels import GridSpec

rig = S.ring_rig(16, (0, 0, 1000), 15000, 4000, 1920, 1080, 1600)
figs = S.place_figures(12, (-8000, -4000), (8000, 4000), seed=0)
t = time.time(); sils, _ = S.render_scene(rig, figs, shade=False); print("scene", time.time() - t)
spec = GridSpec.from_aabb((-9000, -4500, 0), (9000, 4500, 4000), 40.0)
print(spec.dims, spec.num_voxels)
ds = DeviceSilhouettes(rig, sils)
for _ in range(3):
    g = carve_grids(ds, [spec])[0]
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    g = carve_grids(ds, [spec])[0]
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 20
print(f"coarse carve {ms:.3f} ms  -> {spec.num_voxels*16/ms/1e9:.1f} Tvox-proj/s (algorithmic)  ON={g.occupied_count}")
t = time.time(); ref = O.carve(rig, sils, spec.origin, spec.spacing, spec.dims); tc = time.time() - t
print(f"oracle carve {tc:.2f} s ({os.cpu_count()} cpus)  equal={np.array_equal(ref, g.occ)}")
