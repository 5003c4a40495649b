"""GPU busy time vs. wall time of single-stream C3 frames (torch.profiler /
CUPTI kernel records): how much of a frame is host-side bubble, and each
kernel's warm device time inside the replayed frame graph.

    python scripts/frame_gaps.py [--workload C3] [--frames 5]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_1903_11785_b200 import synthetic as S, workloads  # noqa: E402
from paper_1903_11785_b200.executor import executor_for  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="C3")
ap.add_argument("--frames", type=int, default=5)
args = ap.parse_args()
wl = workloads.get(args.workload)
masks, frames = S.render_scene_device(wl.rig, wl.objects(1))
fb = frames.reshape(-1)
foff = np.arange(len(wl.rig), dtype=np.int64) * (frames.shape[1] * frames.shape[2] * 3)
ex = executor_for(wl.cfg, wl.rig)
side = torch.cuda.Stream()  # (not the legacy default stream: frames replay as CUDA graphs)
with torch.cuda.stream(side):
    for _ in range(3):
        ex.run(masks, wl.virtual, fb, foff)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(args.frames):
            ex.run(masks, wl.virtual, fb, foff)
        torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type.name == "CUDA"]
ks = sorted((e.time_range.start, e.time_range.end, e.name) for e in ev)
t0, t1 = ks[0][0], max(k[1] for k in ks)
busy, cur_s, cur_e = 0.0, None, None
for s, e, _ in ks:
    if cur_e is None or s > cur_e:
        if cur_e is not None:
            busy += cur_e - cur_s
        cur_s, cur_e = s, e
    else:
        cur_e = max(cur_e, e)
busy += cur_e - cur_s
gaps = sorted(((ks[i + 1][0] - ks[i][1]), ks[i][2][:40], ks[i + 1][2][:40])
              for i in range(len(ks) - 1))[::-1]
print(f"{len(ks) / args.frames:.0f} GPU records/frame; wall {(t1 - t0) / args.frames:.1f} us/frame, "
      f"busy {busy / args.frames:.1f} us/frame ({busy / (t1 - t0):.1%})")
per = {}
for s_, e_, n_ in ks:
    k = n_.split("(")[0].replace("void ", "")[:48]
    per.setdefault(k, []).append(e_ - s_)
print("per-kernel device time (us/frame, warm, in-graph):")
for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
    n = max(1, round(len(v) / args.frames))
    each = [round(sum(v[i::n]) / args.frames, 1) for i in range(n)] if n > 1 else ""
    print(f"  {sum(v) / args.frames:8.1f}  x{len(v) / args.frames:4.1f}  {k} {each}")
print("largest gaps (us):")
for g, a, b in gaps[:12]:
    print(f"  {g:7.1f}  {a} -> {b}")
