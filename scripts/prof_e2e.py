"""Host-side profile of the e2e path (pipeline.run_sequence), C3 workload."""
import cProfile, pstats, sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1903_11785_b200 import workloads, synthetic as S
from paper_1903_11785_b200.pipeline import run_sequence
wl = workloads.get("C3"); cams = list(wl.rig)
host = []
for f in range(2):
    masks, frames = S.render_scene_device(wl.rig, wl.objects(f))
    m_h = masks.cpu().pin_memory(); f_h = frames.cpu().pin_memory()
    host.append((m_h, {c.id: f_h[k] for k, c in enumerate(cams)}))
def run(n):
    fr = [host[i % 2][1] for i in range(n)]; ms = [host[i % 2][0] for i in range(n)]
    for b, img in run_sequence(wl.cfg, wl.rig, fr, ms, wl.virtual):
        b.merged_mesh.triangles
run(3); torch.cuda.synchronize()
t = time.perf_counter(); run(20); torch.cuda.synchronize(); print("e2e ms/frame", (time.perf_counter() - t) / 20 * 1e3)
pr = cProfile.Profile(); pr.enable(); run(10); torch.cuda.synchronize(); pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(15)
