"""One C3 frame through the native executor between cudaProfilerStart/Stop,
after warm-up frames, for `ncu --profile-from-start off` captures of every
kernel of a frame (launch lists and --set full executed-work counters).

    python scripts/profile_frame.py [--workload C3] [--warm 3] [--frames 1]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1903_11785_b200 import synthetic as S, workloads  # noqa: E402
from paper_1903_11785_b200.executor import executor_for  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="C3")
ap.add_argument("--warm", type=int, default=3)
ap.add_argument("--frames", type=int, default=1)
args = ap.parse_args()
wl = workloads.get(args.workload)
masks, frames = S.render_scene_device(wl.rig, wl.objects(1))
fb = frames.reshape(-1)
foff = np.arange(len(wl.rig), dtype=np.int64) * (frames.shape[1] * frames.shape[2] * 3)
ex = executor_for(wl.cfg, wl.rig)
side = torch.cuda.Stream()  # frames replay as captured graphs after the warm-up
with torch.cuda.stream(side):
    for _ in range(args.warm):
        ex.run(masks, wl.virtual, fb, foff)
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    for _ in range(args.frames):
        out = ex.run(masks, wl.virtual, fb, foff)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
print({k: int(out.stats_raw[k]) for k in ("sparse_tests", "dense_tests", "triangles", "vertices")},
      [round(float(x), 4) for x in out.stats_raw["ms"]])
