"""Where e2e time goes: run_sequence throughput (C3, 4 lanes) with parts of
the host path switched off. python scripts/e2e_probe.py [steps]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1903_11785_b200 import synthetic as S, workloads  # noqa: E402
from paper_1903_11785_b200.pipeline import run_sequence  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 200
lanes = int(os.environ.get("LANES", "4"))
wl = workloads.get("C3")
cams = list(wl.rig)
dev, host = [], []
for f in range(4):
    m, fr = S.render_scene_device(wl.rig, wl.objects(f))
    dev.append((m, {c.id: fr[k] for k, c in enumerate(cams)}))
    mh, fh = m.cpu().pin_memory(), fr.cpu().pin_memory()
    host.append((mh, {c.id: fh[k] for k, c in enumerate(cams)}))


def run(name, src, virt, consume=True):
    def go(n):
        fr = [src[(i + i // lanes) % 4][1] for i in range(n)]
        ms = [src[(i + i // lanes) % 4][0] for i in range(n)]
        for b, img in run_sequence(wl.cfg, wl.rig, fr, ms, virt, lanes=lanes):
            if consume:
                b.merged_mesh.vertices.shape
    go(16)
    torch.cuda.synchronize()
    t = time.perf_counter()
    c0 = time.process_time()
    go(steps)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    print(f"{name:40s} {steps / dt:8.1f} frames/s  host CPU {1e3 * (time.process_time() - c0) / steps:.2f} ms/frame", flush=True)


run("A full (pinned sils, zero-copy colour)", host, wl.virtual)
run("B device sils, zero-copy colour", [(d[0], h[1]) for d, h in zip(dev, host)], wl.virtual)
run("C pinned sils, no colour pass", host, None)
run("D device sils, no colour pass", dev, None)
run("E device sils + device frames", dev, wl.virtual)
