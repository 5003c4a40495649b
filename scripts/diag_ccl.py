"""Time fvv_ccl26 on a C3 coarse grid (warm, CUDA events)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1903_11785_b200 import workloads, synthetic as S
from paper_1903_11785_b200._device import DeviceSilhouettes
from paper_1903_11785_b200.hull import carve_grids, label_grid_async, finish_labels
wl = workloads.get("C3")
masks, _ = S.render_scene_device(wl.rig, wl.objects(0))
ds = DeviceSilhouettes(wl.rig, masks)
g = carve_grids(ds, [wl.cfg.coarse_spec()], 1)[0]
for _ in range(3):
    lab = finish_labels(g, *label_grid_async(g))
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(50):
    label_grid_async(g)
b.record(); torch.cuda.synchronize()
print(f"fvv_ccl26 (coarse C3 grid, {g.spec.num_voxels} voxels, {len(lab.components)} comps): "
      f"{a.elapsed_time(b) / 50 * 1e3:.1f} us/call")
