"""Carve work statistics of one C3 frame's B-1 stage grid and B-3 ROI grids:
tiles culled, foreground / mixed (tile, camera) pairs, and how many voxels
the certified FP32 pass left to the float64 queue.

    python scripts/carve_stats.py [--workload C3]
"""
import argparse
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1903_11785_b200 import _lib, synthetic as S, workloads  # noqa: E402
from paper_1903_11785_b200._device import DeviceSilhouettes, grid_table, stream_handle, words_for  # noqa: E402
from paper_1903_11785_b200.hull import carve, extract_rois, filter_noise, label_components  # noqa: E402
from paper_1903_11785_b200.voxels import GridSpec  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="C3")
args = ap.parse_args()
wl = workloads.get(args.workload)
masks, _ = S.render_scene_device(wl.rig, wl.objects(0))
ds = DeviceSilhouettes(wl.rig, masks)
cfg = wl.cfg
coarse = cfg.coarse_spec()
grid = carve(wl.rig, masks, coarse)
lab = label_components(grid)
_, flab = filter_noise(grid, lab, cfg.noise_params)
rois = extract_rois(flab, coarse, cfg.roi_margin)
fine = [GridSpec.from_aabb(r.lo, r.hi, cfg.fine_spacing) for r in rois]
lib = _lib.load()
ws_bytes = int(lib.fvv_carve_workspace_bytes(_lib.host_ptr(ds.cams), ctypes.c_int(ds.ncam)))
H, W = wl.rig[0].image_height, wl.rig[0].image_width
cells = len(wl.rig) * ((H + 7) >> 3) * ((((W + 7) >> 3) + 31) >> 5)
aff = 96 * 128 * 64
amb_off = aff + 256 + ((8 * cells + 255) & ~255)
for name, specs in (("B-1 stage grid", [coarse]), ("B-3 ROI grids", fine)):
    words = [words_for(s.num_voxels) for s in specs]
    off = np.zeros(len(specs), dtype=np.int64)
    off[1:] = np.cumsum(words)[:-1]
    bits = torch.empty(int(sum(words)), dtype=torch.int32, device="cuda")
    counts = torch.zeros(len(specs), dtype=torch.int64, device="cuda")
    ws = torch.zeros(ws_bytes, dtype=torch.uint8, device="cuda")
    _lib.call("fvv_carve", _lib.host_ptr(ds.cams), ctypes.c_int(ds.ncam), _lib.dev_ptr(ds.bits),
              _lib.host_ptr(ds.word_off), _lib.host_ptr(grid_table(specs)),
              ctypes.c_int(len(specs)), _lib.host_ptr(off), ctypes.c_int(cfg.min_views),
              _lib.dev_ptr(bits), _lib.dev_ptr(counts), _lib.dev_ptr(ws), ctypes.c_size_t(ws_bytes),
              stream_handle())
    torch.cuda.synchronize()
    st = ws[aff:aff + 48].view(torch.int64).cpu().numpy()
    amb = int(ws[amb_off:amb_off + 8].view(torch.int64).cpu().numpy()[0])
    nvox = sum(s.num_voxels for s in specs)
    print(f"{name}: {nvox} voxels, culled tiles {st[0]}, fg (tile,cam) {st[1]}, "
          f"mixed (tile,cam) {st[2]}; octants culled {st[3]}, carved {st[4]} with {st[5]} "
          f"mixed cameras; float64-queued voxels {amb}, ON {int(counts.sum())}")
