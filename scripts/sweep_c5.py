"""C5 kernel sweep (BASELINE.json configs[4]): carve + CCL of a
true n x n x n stage grid, n = 64..1024 (1024^3 lifts the reference's 400 M
voxel budget explicitly), for camera counts 4..64, against the FP32
voxel-projection ceiling. tests/test_gpu_c5.py checks the same grids bit for
bit against the oracle at n = 512 and 1024.

    python scripts/sweep_c5.py [--out profiles/r2_c5_sweep.csv]

Ring rigs of 1080p cameras around 12 C3 figures placed inside the cube; per
(n, cams): device ms of fvv_carve (B-1 semantics, one grid) and fvv_ccl26,
algorithmic voxel-projections/s and the fraction of 148 x 128 x 2 x 1965 MHz
/ 26 FLOP (2.86 T/s).
"""
import argparse, csv, ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1903_11785_b200 import synthetic as S, _lib
from paper_1903_11785_b200._device import DeviceSilhouettes, stream_handle, grid_table
from paper_1903_11785_b200.hull import carve_grids, label_grid_async, finish_labels
from paper_1903_11785_b200.voxels import GridSpec

ap = argparse.ArgumentParser()
ap.add_argument("--out", default="gpurun_out/r2_c5_sweep.csv")
ap.add_argument("--sizes", default="64,128,256,512,1024")
ap.add_argument("--cams", default="4,8,16,32,64")
args = ap.parse_args()
props = torch.cuda.get_device_properties(0)
ceiling = props.multi_processor_count * 128 * 2 * 1965e6 / 26
rows = []
side = 8000.0
objs = S.place_figures(12, (-3000, -3000), (3000, 3000), seed=0)  # as tests/test_gpu_c5.py
for ncam in [int(c) for c in args.cams.split(",")]:
    rig = S.ring_rig(ncam, (0, 0, 1000), 15000, 4000, 1920, 1080, 1600)
    masks, _ = S.render_scene_device(rig, objs)
    ds = DeviceSilhouettes(rig, masks)
    for n in [int(s) for s in args.sizes.split(",")]:
        spec = GridSpec(origin=(-side / 2, -side / 2, 0.0), spacing=side / n, dims=(n, n, n),
                        budget=n ** 3)
        for _ in range(2):
            g = carve_grids(ds, [spec], 1)[0]
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 10
        a.record()
        for _ in range(reps):
            g = carve_grids(ds, [spec], 1)[0]
        b.record(); torch.cuda.synchronize()
        carve_ms = a.elapsed_time(b) / reps
        lab = finish_labels(g, *label_grid_async(g))
        a.record()
        for _ in range(reps):
            label_grid_async(g)
        b.record(); torch.cuda.synchronize()
        ccl_ms = a.elapsed_time(b) / reps
        proj = spec.num_voxels * ncam
        rate = proj / (carve_ms / 1e3)
        row = {"n": n, "dims": f"{n}x{n}x{n}", "cams": ncam, "voxels": spec.num_voxels,
               "occupied": int(g.occupied_count), "components": len(lab.components),
               "carve_ms": round(carve_ms, 4), "T_voxel_proj_per_s": round(rate / 1e12, 4),
               "frac_fp32_ceiling": round(rate / ceiling, 4), "ccl_ms": round(ccl_ms, 4),
               "ccl_GBps": round((spec.num_voxels / 8 + 4 * spec.num_voxels) / (ccl_ms / 1e3) / 1e9, 2)}
        rows.append(row)
        print(row, flush=True)
os.makedirs(os.path.dirname(args.out) or ".", exist_ok=True)
with open(args.out, "w", newline="") as fh:
    w = csv.DictWriter(fh, fieldnames=list(rows[0]))
    w.writeheader()
    w.writerows(rows)
