"""Host-side cost of one single-stream C3 frame through FrameExecutor.run:
wall time per frame, the time inside the native fvv_frame_run call (bind +
graph launch + wait + result reads) and the Python around it.

    python scripts/run_overhead.py [--frames 200]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1903_11785_b200 import _lib, synthetic as S, workloads  # noqa: E402
from paper_1903_11785_b200.executor import executor_for  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--frames", type=int, default=200)
ap.add_argument("--no-stage-times", action="store_true",
                help="skip the per-stage event readout (FrameExecutor.stage_times)")
args = ap.parse_args()
wl = workloads.get("C3")
masks, frames = S.render_scene_device(wl.rig, wl.objects(1))
fb = frames.reshape(-1)
foff = np.arange(len(wl.rig), dtype=np.int64) * (frames.shape[1] * frames.shape[2] * 3)
ex = executor_for(wl.cfg, wl.rig)
ex.stage_times = not args.no_stage_times
lib = _lib.load()
native = {"t": 0.0}
orig = lib.fvv_frame_run


def timed_run(*a):
    t = time.perf_counter()
    r = orig(*a)
    native["t"] += time.perf_counter() - t
    return r


side = torch.cuda.Stream()
with torch.cuda.stream(side):
    for _ in range(10):
        ex.run(masks, wl.virtual, fb, foff)
    torch.cuda.synchronize()
    lib.fvv_frame_run = timed_run
    t0 = time.perf_counter()
    for _ in range(args.frames):
        out = ex.run(masks, wl.virtual, fb, foff)
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) / args.frames * 1e6
lib.fvv_frame_run = orig
ms = float(np.sum(out.stats_raw["ms"][:7]))  # (0 without stage times)
print(f"wall {wall:.1f} us/frame, native call {native['t'] / args.frames * 1e6:.1f} us, "
      f"python {wall - native['t'] / args.frames * 1e6:.1f} us, device stages {ms * 1e3:.1f} us")
