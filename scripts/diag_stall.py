"""Find start-of-sequence stalls in run_sequence: timestamped trace of the
first frames of repeated calls."""
import sys, os, time, gc, threading
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1903_11785_b200 import workloads, synthetic as S, pipeline as P, executor as E
wl = workloads.get("C3"); cams = list(wl.rig)
host = []
for f in range(4):
    masks, frames = S.render_scene_device(wl.rig, wl.objects(f), shade=True)
    host.append((masks.cpu().pin_memory(), {c.id: t for c, t in zip(cams, frames.cpu().pin_memory())}))
LOG = []
T0 = [0.0]
def tr(name, fn):
    def g(*a, **k):
        t = time.perf_counter(); r = fn(*a, **k); e = time.perf_counter()
        if e - t > 0.003: LOG.append(f"  {threading.current_thread().name}: {name} {1e3*(t-T0[0]):.1f}+{1e3*(e-t):.1f} ms")
        return r
    return g
E.FrameExecutor.run = tr("run", E.FrameExecutor.run)
E.FrameOutput.to_host_async = tr("to_host_async", E.FrameOutput.to_host_async)
P._prefetch = tr("prefetch", P._prefetch)
P.bundle_from_output = tr("bundle", P.bundle_from_output)
E.executor_for = tr("executor_for", E.executor_for)
torch.cuda.Stream.__init__ = tr("Stream()", torch.cuda.Stream.__init__) if False else torch.cuda.Stream.__init__
gc.callbacks.append(lambda phase, info: LOG.append(f"  gc {phase} gen{info['generation']} {1e3*(time.perf_counter()-T0[0]):.1f}"))
def run(n, label):
    fr = [host[i % 4][1] for i in range(n)]; ms = [host[i % 4][0] for i in range(n)]
    LOG.clear()
    torch.cuda.synchronize(); T0[0] = t0 = time.perf_counter(); ts = []
    for b, img in P.run_sequence(wl.cfg, wl.rig, fr, ms, wl.virtual):
        b.merged_mesh.object_ids; ts.append(time.perf_counter())
    torch.cuda.synchronize(); t1 = time.perf_counter()
    d = np.diff([t0] + ts) * 1e3
    print(f"{label}: {(t1 - t0) / n * 1e3:.2f} ms/frame; first intervals: " + " ".join(f"{x:.1f}" for x in d[:6]))
    for l in LOG[:30]: print(l)
for r in range(6):
    run(30 if r else 12, f"call{r}")
