import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1903_11785_b200 import workloads, synthetic as S
from paper_1903_11785_b200.pipeline import run_sequence
wl = workloads.get("C3"); cams = list(wl.rig)
host = []
for f in range(4):
    masks, frames = S.render_scene_device(wl.rig, wl.objects(f))
    host.append((masks.cpu().pin_memory(), {c.id: t for c, t in zip(cams, frames.cpu().pin_memory())}))
for rep in range(3):
    fr = [host[i % 4][1] for i in range(30)]; ms = [host[i % 4][0] for i in range(30)]
    torch.cuda.synchronize(); t0 = time.perf_counter(); ts = []
    for b, img in run_sequence(wl.cfg, wl.rig, fr, ms, wl.virtual):
        b.merged_mesh.triangles; ts.append(time.perf_counter())
    torch.cuda.synchronize(); t1 = time.perf_counter()
    d = [ (ts[i] - (ts[i-1] if i else t0)) * 1e3 for i in range(len(ts))]
    print(f"rep {rep}: {((t1-t0)/30)*1e3:.2f} ms/frame; per-frame ms: " + " ".join(f"{x:.1f}" for x in d))
