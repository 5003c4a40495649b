"""GPU timeline of run_sequence's three streams (H2D / compute / D2H), C3."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import numpy as np
STG = []
from paper_1903_11785_b200 import workloads, synthetic as S, pipeline as P
wl = workloads.get("C3"); cams = list(wl.rig)
host = []
for f in range(4):
    masks, frames = S.render_scene_device(wl.rig, wl.objects(f))
    host.append((masks.cpu().pin_memory(), {c.id: t for c, t in zip(cams, frames.cpu().pin_memory())}))
# H2D / D2H raw bandwidth
big = torch.empty(132710400, dtype=torch.uint8).pin_memory(); d = torch.empty_like(big, device="cuda")
for _ in range(3): d.copy_(big, non_blocking=True)
torch.cuda.synchronize(); t = time.perf_counter()
for _ in range(10): d.copy_(big, non_blocking=True)
torch.cuda.synchronize(); print("H2D GB/s", 10 * big.numel() / (time.perf_counter() - t) / 1e9)
t = time.perf_counter()
for _ in range(10): big.copy_(d, non_blocking=True)
torch.cuda.synchronize(); print("D2H GB/s", 10 * big.numel() / (time.perf_counter() - t) / 1e9)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream(); h2 = torch.empty(38157678, dtype=torch.uint8).pin_memory()
torch.cuda.synchronize(); t = time.perf_counter()
for _ in range(10):
    with torch.cuda.stream(s1): d.copy_(big, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d[:h2.numel()], non_blocking=True)
torch.cuda.synchronize(); print("duplex H2D+D2H ms/iter", (time.perf_counter() - t) / 10 * 1e3)

# instrumented loop
import paper_1903_11785_b200.executor as E
T = {"run": 0.0, "to_host": 0.0, "finish": 0.0, "prefetch": 0.0, "wait": 0.0}
orig_run, orig_th, orig_pf = E.FrameExecutor.run, E.FrameOutput.to_host_async, P._prefetch
def wrap(name, fn):
    def g(*a, **k):
        t = time.perf_counter(); r = fn(*a, **k); T[name] += time.perf_counter() - t; return r
    return g
T["gpu_ms"] = 0.0
from paper_1903_11785_b200 import _lib as L
_lib_h = L.load(); _orig_fr = _lib_h.fvv_frame_run; T["c_run"] = 0.0
def _fr(*a):
    t = time.perf_counter(); r = _orig_fr(*a); T["c_run"] += time.perf_counter() - t; return r
_lib_h.fvv_frame_run = _fr
def run_w(*a, **k):
    t = time.perf_counter(); r = orig_run(*a, **k); T["run"] += time.perf_counter() - t
    T["gpu_ms"] += float(r.stats_raw["ms"][:8].sum()) / 1e3
    STG.append(np.array(r.stats_raw["ms"][:8], dtype=np.float64))
    return r
E.FrameExecutor.run = run_w; E.FrameOutput.to_host_async = wrap("to_host", orig_th)
P._prefetch = wrap("prefetch", orig_pf)
orig_g = P._gather_to_device
T["gather"] = 0.0
P._gather_to_device = wrap("gather", orig_g)
orig_hp = P._host_piece; T["piece"] = 0.0
P._host_piece = wrap("piece", orig_hp)
orig_bfo = P.bundle_from_output; P.bundle_from_output = wrap("finish", orig_bfo)
for rep in range(2):
    for k in T: T[k] = 0.0
    fr = [host[i % 4][1] for i in range(30)]; ms = [host[i % 4][0] for i in range(30)]
    torch.cuda.synchronize(); t0 = time.perf_counter(); tl = 0.0
    g = P.run_sequence(wl.cfg, wl.rig, fr, ms, wl.virtual)
    for b, img in g:
        b.merged_mesh.triangles
    torch.cuda.synchronize(); el = time.perf_counter() - t0
    print("stage ms:", np.round(np.mean(STG[-25:], axis=0), 3))
    print(f"rep {rep}: {el/30*1e3:.2f} ms/frame; " + " ".join(f"{k}={v/30*1e3:.2f}" for k, v in T.items()))
