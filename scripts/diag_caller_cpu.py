"""CPU time (thread_time) of the caller-side pieces of run_sequence per frame:
input staging (_prefetch), SceneBundle assembly, the consumer; plus the
worker-side executor.run wrapper. C3, 4 lanes, pinned host inputs."""
import collections
import gc
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1903_11785_b200 import executor as E, pipeline as P, synthetic as S, workloads

ACC = collections.defaultdict(float)
CNT = collections.Counter()


def timed(name, fn):
    def w(*a, **k):
        t = time.thread_time()
        try:
            return fn(*a, **k)
        finally:
            ACC[name] += time.thread_time() - t
            CNT[name] += 1
    return w


P._prefetch = timed("_prefetch", P._prefetch)
P.bundle_from_output = timed("bundle_from_output", P.bundle_from_output)
E.FrameExecutor.run = timed("executor.run (worker)", E.FrameExecutor.run)
E.FrameOutput.to_host_async = timed("to_host_async (worker)", E.FrameOutput.to_host_async)
E.HostBlock.arrays = timed("HostBlock.arrays", E.HostBlock.arrays)

wl = workloads.get("C3")
cams = list(wl.rig)
host = []
for f in range(4):
    masks, frames = S.render_scene_device(wl.rig, wl.objects(f), shade=True)
    host.append((masks.cpu().pin_memory(), {c.id: t for c, t in zip(cams, frames.cpu().pin_memory())}))


def run(n):
    fr = [host[i % 4][1] for i in range(n)]
    ms = [host[i % 4][0] for i in range(n)]
    for b, img in P.run_sequence(wl.cfg, wl.rig, fr, ms, wl.virtual, lanes=4):
        b.merged_mesh.vertices.shape, b.merged_mesh.triangles.shape, img.color.shape


run(12)
torch.cuda.synchronize()
ACC.clear(); CNT.clear()
gc.collect(); gc.disable()
t0, c0 = time.perf_counter(), time.thread_time()
run(80)
torch.cuda.synchronize()
dt = time.perf_counter() - t0
print(f"{dt / 80 * 1e3:.3f} ms/frame wall; caller thread CPU {(time.thread_time() - c0) / 80 * 1e3:.3f} ms/frame")
for k, v in sorted(ACC.items(), key=lambda kv: -kv[1]):
    print(f"  {k:28s} {v / 80 * 1e3:7.3f} ms/frame  ({CNT[k]} calls)")
