"""BASELINE.json workload definitions: rigs, scenes,
pipeline configs and the virtual viewpoint of each config.

  C1 8 cams 640x480, 3 ellipsoids, 128^3 coarse (31.25 mm), 12.5 mm fine
  C2 judo: 16 cams 1080p, 8x8 m mat, 2 figures, 40 mm / 5 mm
  C3 volleyball: 16 cams 1080p, 18x9 m court, 12 figures, 40 mm / 10 mm
  C4 volleyball at 4K: 32 cams 3840x2160, 5 mm ROI voxels
Frame f animates every figure at t = f / 30 s (positions from rng(0)).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import synthetic as S
from .pipeline import PipelineConfig


@dataclass
class Workload:
    name: str
    rig: object
    cfg: PipelineConfig
    virtual: object
    n_figures: int
    area_lo: tuple
    area_hi: tuple
    description: str

    def objects(self, frame: int = 0):
        if self.name == "C1":
            return c1_objects(frame)
        return S.place_figures(self.n_figures, self.area_lo, self.area_hi, seed=0,
                               t=frame / 30.0)


def c1_objects(frame: int = 0):
    yaw = 0.15 * np.sin(2 * np.pi * frame / 30.0)
    out = []
    for (x, y), a in zip(((-900.0, -500.0), (800.0, 600.0), (300.0, -1100.0)), (0.3, -0.7, 1.2)):
        c, s = np.cos(a + yaw), np.sin(a + yaw)
        rot = np.array([[c, -s, 0.0], [s, c, 0.0], [0.0, 0.0, 1.0]])
        out.append(S.Ellipsoid((x, y, 900.0), (450.0, 350.0, 850.0), rot,
                               np.array([190.0, 110.0, 80.0])))
    return out


def _virtual_on_ring(cam_id, target, radius, height, width, img_h, focal, angle_deg):
    ang = np.deg2rad(angle_deg)
    target = np.asarray(target, dtype=np.float64)
    pos = target + np.array([radius * np.cos(ang), radius * np.sin(ang), height])
    return S.look_at_camera(cam_id, pos, target, width, img_h, focal)


def get(name: str) -> Workload:
    if name == "C1":
        rig = S.ring_rig(8, (0, 0, 900), 6000, 2000, 640, 480, 520)
        cfg = PipelineConfig(stage_lo=(-2000, -2000, 0), stage_hi=(2000, 2000, 4000),
                             coarse_spacing=31.25, fine_spacing=12.5, t_small=3)
        virt = _virtual_on_ring(100, (0, 0, 900), 6000, 2000, 640, 480, 520, 22.5)
        return Workload("C1", rig, cfg, virt, 3, (-1500, -1500), (1500, 1500),
                        "8 cams 640x480, 3 ellipsoids, 128^3 coarse / 12.5 mm fine")
    if name == "C2":
        rig = S.ring_rig(16, (0, 0, 900), 9000, 3000, 1920, 1080, 1500)
        cfg = PipelineConfig(stage_lo=(-4000, -4000, 0), stage_hi=(4000, 4000, 2500),
                             coarse_spacing=40.0, fine_spacing=5.0)
        virt = _virtual_on_ring(100, (0, 0, 900), 9000, 3000, 1920, 1080, 1500, 11.25)
        return Workload("C2", rig, cfg, virt, 2, (-1500, -1500), (1500, 1500),
                        "judo: 16 cams 1080p, 2 figures, 40 mm / 5 mm")
    if name in ("C3", "C4"):
        n, w, h, f = (16, 1920, 1080, 1600) if name == "C3" else (32, 3840, 2160, 3200)
        rig = S.ring_rig(n, (0, 0, 1000), 15000, 4000, w, h, f)
        cfg = PipelineConfig(stage_lo=(-9000, -4500, 0), stage_hi=(9000, 4500, 4000),
                             coarse_spacing=40.0, fine_spacing=10.0 if name == "C3" else 5.0)
        virt = _virtual_on_ring(100, (0, 0, 1000), 15000, 4000, 1920, 1080, 1600, 11.25)
        desc = ("volleyball: 16 cams 1920x1080, 12 figures, 40 mm coarse / 10 mm ROI"
                if name == "C3" else "volleyball 4K: 32 cams 3840x2160, 12 figures, 5 mm ROI")
        return Workload(name, rig, cfg, virt, 12, (-8000, -3800), (8000, 3800), desc)
    raise ValueError(f"unknown workload {name!r}")
