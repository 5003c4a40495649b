"""Single-stream C3 frames with the virtual viewpoint moving every frame
(a camera path, the usual free-viewpoint case) against a fixed viewpoint:
frames per second through FrameExecutor.run.

    python scripts/moving_view.py [--frames 120]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1903_11785_b200 import synthetic as S, workloads  # noqa: E402
from paper_1903_11785_b200.executor import executor_for  # noqa: E402
from paper_1903_11785_b200.workloads import _virtual_on_ring  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--frames", type=int, default=120)
args = ap.parse_args()
wl = workloads.get("C3")
masks, frames = S.render_scene_device(wl.rig, wl.objects(1))
fb = frames.reshape(-1)
foff = np.arange(len(wl.rig), dtype=np.int64) * (frames.shape[1] * frames.shape[2] * 3)
path = [_virtual_on_ring(100, (0, 0, 1000), 15000, 4000, 1920, 1080, 1600, 11.25 + 0.5 * k)
        for k in range(args.frames)]
ex = executor_for(wl.cfg, wl.rig)
ex.stage_times = False
side = torch.cuda.Stream()
with torch.cuda.stream(side):
    for _ in range(6):
        ex.run(masks, wl.virtual, fb, foff)
    torch.cuda.synchronize()
    for name, views in (("fixed", [wl.virtual] * args.frames), ("moving", path)):
        t = time.perf_counter()
        for v in views:
            ex.run(masks, v, fb, foff)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t
        print(f"{name}: {args.frames / dt:.1f} frames/s (last mode {ex.last_mode})")
