"""Render-stage GPU time with colour frames sampled in place from pinned host
memory (zero-copy) vs. frames resident on the device (C3, one lane)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1903_11785_b200 import synthetic as S, workloads
from paper_1903_11785_b200 import pipeline as P
from paper_1903_11785_b200.pipeline import run_sequence

MS = []
_orig = P.bundle_from_output


def _record(out, *a, **k):
    MS.append([round(float(x), 3) for x in out.stats_raw["ms"][:7]])
    return _orig(out, *a, **k)


P.bundle_from_output = _record

wl = workloads.get("C3")
cams = list(wl.rig)
masks, frames = S.render_scene_device(wl.rig, wl.objects(0), shade=True)
pinned = {c.id: t for c, t in zip(cams, frames.cpu().pin_memory())}
device = {c.id: t for c, t in zip(cams, frames)}
m_host = masks.cpu().pin_memory()
for name, fr in (("zero-copy", pinned), ("device", device)):
    MS.clear()
    for b, img in run_sequence(wl.cfg, wl.rig, [fr] * 12, [m_host] * 12, wl.virtual, lanes=1):
        pass
    print(name, "stage ms B-1 B-2 B-3 C D-1 D-2 E (last 4 frames):", MS[-4:])
