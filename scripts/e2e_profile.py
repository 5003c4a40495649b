"""cProfile of the caller thread of pipeline.run_sequence (C3, 8 lanes, pinned
host inputs): where the Python side of the e2e path spends its time.

    python scripts/e2e_profile.py
"""
import cProfile, pstats, os, sys, io
sys.path.insert(0, os.getcwd())
import torch, numpy as np
from paper_1903_11785_b200 import synthetic as S, workloads
from paper_1903_11785_b200.pipeline import run_sequence
wl = workloads.get("C3")
host = []
for f in range(4):
    m, fr = S.render_scene_device(wl.rig, wl.objects(f))
    host.append((m.cpu().pin_memory(), {c.id: t for c, t in zip(wl.rig, fr.cpu().pin_memory())}))
def consume(b, img):
    n = 0
    if b is not None:
        m = b.merged_mesh; n += m.vertices.shape[0] + m.triangles.shape[0]
    if img is not None: n += img.color.shape[0]
    return n
def run(n):
    fr = [host[i % 4][1] for i in range(n)]; ms = [host[i % 4][0] for i in range(n)]
    for b, img in run_sequence(wl.cfg, wl.rig, fr, ms, wl.virtual, lanes=8):
        consume(b, img)
run(120); torch.cuda.synchronize()
pr = cProfile.Profile(); pr.enable(); run(400); torch.cuda.synchronize(); pr.disable()
s = io.StringIO(); pstats.Stats(pr, stream=s).sort_stats("tottime").print_stats(22); print(s.getvalue()[:4000])
