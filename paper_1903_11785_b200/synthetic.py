"""Synthetic multi-camera scenes (test and benchmark harness, not hot path).

The rig helpers restate the reference's ``look_at_camera`` / ``ring_rig``
(synthetic.py:111-162) so rigs are identical to the reference's. The scene
primitives add what BASELINE.json's workloads need and the reference lacks:
an ``Ellipsoid`` (centre, semi-axes, orientation) and an articulated
``Figure`` (11 ellipsoid parts with sinusoidal joint angles). Silhouettes
are exact per-pixel ray casts (pixel centre ray hits any part) and frames
are Lambertian-shaded like the reference's ``shade_frame``
(synthetic.py:195-218). Both are INPUTS: the parity tests feed the same
arrays to the GPU path and to the CPU oracle.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .camera import CameraModel, CameraRig

BG_COLOR = np.array([32, 36, 40], dtype=np.float64)
AMBIENT = 0.35
LIGHT_DIR = np.array([0.3, 0.5, -0.8]) / np.linalg.norm([0.3, 0.5, -0.8])


def look_at_camera(cam_id, center, target, width, height, focal) -> CameraModel:
    """Zero-distortion camera at ``center`` aimed at ``target``, z up."""
    center = np.asarray(center, dtype=np.float64)
    target = np.asarray(target, dtype=np.float64)
    fwd = target - center
    fwd = fwd / np.linalg.norm(fwd)
    up = np.array([0.0, 0.0, 1.0])
    if abs(fwd @ up) > 0.999:
        up = np.array([0.0, 1.0, 0.0])
    right = np.cross(fwd, up)
    right /= np.linalg.norm(right)
    down = np.cross(fwd, right)
    rot = np.stack([right, down, fwd])
    return CameraModel(id=cam_id, image_width=width, image_height=height, fx=focal, fy=focal,
                       cx=(width - 1) / 2.0, cy=(height - 1) / 2.0, rotation=rot,
                       translation=-rot @ center)


def ring_rig(n_cameras, target, ring_radius, height, width=1920, image_height=1080,
             focal=1200.0) -> CameraRig:
    """``n_cameras`` on a horizontal ring around ``target``, all aimed at it."""
    target = np.asarray(target, dtype=np.float64)
    cams = []
    for i in range(n_cameras):
        ang = 2.0 * np.pi * i / n_cameras
        pos = target + np.array([ring_radius * np.cos(ang), ring_radius * np.sin(ang), height])
        cams.append(look_at_camera(i, pos, target, width, image_height, focal))
    return CameraRig(cams)


def _rot_z(yaw):
    c, s = np.cos(yaw), np.sin(yaw)
    return np.array([[c, -s, 0.0], [s, c, 0.0], [0.0, 0.0, 1.0]])


def _frame_along(direction):
    """Orthonormal basis whose third column is ``direction``."""
    d = np.asarray(direction, dtype=np.float64)
    d = d / np.linalg.norm(d)
    helper = np.array([1.0, 0.0, 0.0]) if abs(d[0]) < 0.9 else np.array([0.0, 1.0, 0.0])
    a = np.cross(helper, d)
    a /= np.linalg.norm(a)
    b = np.cross(d, a)
    return np.stack([a, b, d], axis=1)


@dataclass
class Ellipsoid:
    """Solid ellipsoid: |Q^T (p - c) / s| <= 1 (Q's columns = world axes)."""

    center: np.ndarray
    semi_axes: tuple
    orient: np.ndarray = field(default_factory=lambda: np.eye(3))
    color: np.ndarray = field(default_factory=lambda: np.array([190.0, 120.0, 90.0]))

    def __post_init__(self):
        self.center = np.asarray(self.center, dtype=np.float64).reshape(3)
        self.semi_axes = np.asarray(self.semi_axes, dtype=np.float64).reshape(3)
        self.orient = np.asarray(self.orient, dtype=np.float64).reshape(3, 3)
        self.color = np.asarray(self.color, dtype=np.float64).reshape(3)
        if (self.semi_axes <= 0).any():
            raise ValueError("ellipsoid semi-axes must be positive")

    def parts(self):
        return [self]

    def aabb(self):
        half = np.sqrt(((self.orient * self.semi_axes[None, :]) ** 2).sum(axis=1))
        return self.center - half, self.center + half

    def ray_hits(self, origin, dirs):
        """Smallest ray parameter > 1e-9 per ray, +inf on miss."""
        o = ((origin - self.center) @ self.orient) / self.semi_axes
        d = (dirs @ self.orient) / self.semi_axes
        a = (d * d).sum(-1)
        b = d @ o
        c = o @ o - 1.0
        disc = b * b - a * c
        hit = disc >= 0
        sq = np.sqrt(np.where(hit, disc, 0.0))
        t0 = (-b - sq) / a
        t1 = (-b + sq) / a
        t = np.where(t0 > 1e-9, t0, t1)
        return np.where(hit & (t > 1e-9), t, np.inf)

    def normal_at(self, p):
        local = ((p - self.center) @ self.orient) / self.semi_axes ** 2
        n = local @ self.orient.T
        return n / np.linalg.norm(n, axis=-1, keepdims=True)

    def contains(self, pts):
        q = ((np.asarray(pts) - self.center) @ self.orient) / self.semi_axes
        return (q * q).sum(-1) <= 1.0


def _limb(a, b, radius, color):
    a, b = np.asarray(a, float), np.asarray(b, float)
    half = 0.5 * np.linalg.norm(b - a)
    return Ellipsoid(0.5 * (a + b), (radius, radius, half + 0.6 * radius), _frame_along(b - a),
                     color)


@dataclass
class Figure:
    """Articulated 'player': 11 ellipsoid parts (pelvis, torso, head, upper
    and lower arms and legs). Joint angles are sinusoids of ``t`` with
    per-figure phase, so a frame index animates every figure."""

    root: np.ndarray  # floor position (x, y) in mm
    yaw: float = 0.0
    scale: float = 1.0
    phase: float = 0.0
    t: float = 0.0
    color: np.ndarray = field(default_factory=lambda: np.array([200.0, 90.0, 70.0]))

    def parts(self):
        s = self.scale
        w = 2.0 * np.pi * 1.2 * self.t + self.phase
        rz = _rot_z(self.yaw)
        base = np.array([self.root[0], self.root[1], 0.0])

        def P(x, y, z):
            return base + rz @ (s * np.array([x, y, z], dtype=np.float64))

        skin = np.array([225.0, 180.0, 150.0])
        shirt = self.color
        shorts = 0.55 * self.color + 40.0
        swing = 0.55 * np.sin(w)
        parts = [
            Ellipsoid(P(0, 0, 930), (s * 170, s * 115, s * 120), rz, shorts),   # pelvis
            Ellipsoid(P(0, 0, 1300), (s * 200, s * 125, s * 270), rz, shirt),   # torso
            Ellipsoid(P(0, 0, 1720), (s * 100, s * 105, s * 125), rz, skin),    # head
        ]
        for side in (-1.0, 1.0):
            sh = P(side * 235, 0, 1510)
            a_sw = side * swing
            el = sh + rz @ (s * 300 * np.array([side * 0.15, np.sin(a_sw), -np.cos(a_sw)]))
            bend = 0.4 + 0.3 * np.sin(w + 0.8)
            wr = el + rz @ (s * 270 * np.array([0.0, np.sin(a_sw + bend), -np.cos(a_sw + bend)]))
            parts.append(_limb(sh, el, s * 55, shirt))
            parts.append(_limb(el, wr, s * 45, skin))
            hip = P(side * 95, 0, 900)
            l_sw = -side * 0.8 * swing
            kn = hip + rz @ (s * 440 * np.array([0.0, np.sin(l_sw), -np.cos(l_sw)]))
            kb = max(0.0, 0.5 * np.sin(w + side * 1.3))
            an = kn + rz @ (s * 430 * np.array([0.0, np.sin(l_sw - kb), -np.cos(l_sw - kb)]))
            parts.append(_limb(hip, kn, s * 75, shorts))
            parts.append(_limb(kn, an, s * 55, skin))
        return parts


def scene_parts(objects):
    out = []
    for o in objects:
        out.extend(o.parts())
    return out


def _camera_rays(cam, x0, x1, y0, y1):
    us, vs = np.meshgrid(np.arange(x0, x1, dtype=np.float64), np.arange(y0, y1, dtype=np.float64))
    yn = (vs - cam.cy) / cam.fy
    xn = (us - cam.cx) / cam.fx - cam.skew * yn
    d = np.stack([xn, yn, np.ones_like(xn)], axis=-1) @ cam.rotation
    d /= np.linalg.norm(d, axis=-1, keepdims=True)
    return cam.center, d


def _pixel_box(cam, part):
    """Conservative pixel bbox of a part (projected world-AABB corners)."""
    lo, hi = part.aabb()
    corners = np.array([[x, y, z] for x in (lo[0], hi[0]) for y in (lo[1], hi[1])
                        for z in (lo[2], hi[2])])
    pc = corners @ cam.rotation.T + cam.translation
    if (pc[:, 2] <= 1.0).any():
        return 0, cam.image_width, 0, cam.image_height
    u = cam.fx * (pc[:, 0] / pc[:, 2] + cam.skew * pc[:, 1] / pc[:, 2]) + cam.cx
    v = cam.fy * pc[:, 1] / pc[:, 2] + cam.cy
    x0 = int(np.clip(np.floor(u.min()) - 1, 0, cam.image_width))
    x1 = int(np.clip(np.ceil(u.max()) + 2, 0, cam.image_width))
    y0 = int(np.clip(np.floor(v.min()) - 1, 0, cam.image_height))
    y1 = int(np.clip(np.ceil(v.max()) + 2, 0, cam.image_height))
    return x0, x1, y0, y1


def render_camera(cam, objects, shade=True, noise_sigma=0.0, seed=0):
    """(silhouette bool (H,W), frame uint8 (H,W,3) or None) for one camera."""
    parts = scene_parts(objects)
    h, w = cam.image_height, cam.image_width
    depth = np.full((h, w), np.inf)
    owner = np.full((h, w), -1, dtype=np.int32)
    for pi, part in enumerate(parts):
        x0, x1, y0, y1 = _pixel_box(cam, part)
        if x1 <= x0 or y1 <= y0:
            continue
        origin, dirs = _camera_rays(cam, x0, x1, y0, y1)
        t = part.ray_hits(origin, dirs.reshape(-1, 3)).reshape(y1 - y0, x1 - x0)
        sub = depth[y0:y1, x0:x1]
        closer = t < sub
        sub[closer] = t[closer]
        owner[y0:y1, x0:x1][closer] = pi
    sil = np.isfinite(depth)
    if not shade:
        return sil, None
    img = np.broadcast_to(BG_COLOR, (h, w, 3)).copy()
    ys, xs = np.nonzero(sil)
    if len(ys):
        origin, _ = _camera_rays(cam, 0, 1, 0, 1)
        yn = (ys - cam.cy) / cam.fy
        xn = (xs - cam.cx) / cam.fx - cam.skew * yn
        d = np.stack([xn, yn, np.ones_like(xn)], axis=-1) @ cam.rotation
        d /= np.linalg.norm(d, axis=-1, keepdims=True)
        pts = origin + depth[ys, xs, None] * d
        for pi in np.unique(owner[ys, xs]):
            sel = owner[ys, xs] == pi
            n = parts[pi].normal_at(pts[sel])
            lum = AMBIENT + (1.0 - AMBIENT) * np.maximum(0.0, -(n @ LIGHT_DIR))
            img[ys[sel], xs[sel]] = parts[pi].color * lum[:, None]
    if noise_sigma > 0:
        img = img + np.random.default_rng(seed + cam.id).normal(0.0, noise_sigma, img.shape)
    return sil, np.clip(np.rint(img), 0, 255).astype(np.uint8)


def render_scene(rig, objects, shade=True, noise_sigma=0.0, seed=0):
    """Silhouettes (list, rig order) and frames (dict id -> uint8) for a rig."""
    sils, frames = [], {}
    for cam in rig:
        s, f = render_camera(cam, objects, shade, noise_sigma, seed)
        sils.append(s)
        frames[cam.id] = f
    return sils, frames


def place_figures(n, area_lo, area_hi, seed=0, t=0.0, min_gap=1200.0):
    """``n`` figures at non-overlapping random floor positions (rng(seed)),
    animated at time ``t`` (frame f of a 30 fps sequence: t = f / 30)."""
    rng = np.random.default_rng(seed)
    lo, hi = np.asarray(area_lo, float), np.asarray(area_hi, float)
    roots = []
    while len(roots) < n:
        p = rng.uniform(lo, hi)
        if all(np.linalg.norm(p - q) >= min_gap for q in roots):
            roots.append(p)
    palette = [np.array(c, float) for c in ((200, 70, 60), (60, 110, 200), (230, 200, 60),
                                            (70, 170, 90), (150, 80, 190), (240, 140, 50))]
    figs = []
    for i, r in enumerate(roots):
        figs.append(Figure(root=r, yaw=float(rng.uniform(-np.pi, np.pi)),
                           scale=float(rng.uniform(0.9, 1.08)),
                           phase=float(rng.uniform(0, 2 * np.pi)), t=t,
                           color=palette[i % len(palette)]))
    return figs


def parts_table(objects) -> np.ndarray:
    """(P, 18) float64 records for fvv_render_ellipsoids."""
    parts = scene_parts(objects)
    tab = np.zeros((len(parts), 18))
    for i, p in enumerate(parts):
        tab[i, 0:3] = p.center
        tab[i, 3:12] = p.orient.reshape(9)
        tab[i, 12:15] = p.semi_axes
        tab[i, 15:18] = p.color
    return tab


def render_scene_device(rig, objects, shade=True):
    """GPU ray cast of the scene into every rig camera (harness kernel
    fvv_render_ellipsoids). Returns (masks uint8 (N,H,W), frames uint8
    (N,H,W,3) or None) as CUDA tensors; all cameras must share one size."""
    import ctypes

    import torch

    from . import _lib
    from ._device import cam_table, require_cuda, stream_handle

    dev = require_cuda()
    cams = list(rig)
    h, w = cams[0].image_height, cams[0].image_width
    if any((c.image_height, c.image_width) != (h, w) for c in cams):
        raise ValueError("render_scene_device needs equal image sizes")
    tab = torch.from_numpy(np.ascontiguousarray(parts_table(objects))).to(dev)
    masks = torch.empty((len(cams), h, w), dtype=torch.uint8, device=dev)
    frames = torch.empty((len(cams), h, w, 3), dtype=torch.uint8, device=dev) if shade else None
    shading = np.array([AMBIENT, *LIGHT_DIR, *BG_COLOR], dtype=np.float64)
    for i, c in enumerate(cams):
        _lib.call("fvv_render_ellipsoids", _lib.host_ptr(cam_table([c])), _lib.dev_ptr(tab),
                  ctypes.c_int(len(tab)), _lib.dev_ptr(masks[i]),
                  _lib.dev_ptr(frames[i]) if shade else ctypes.c_void_p(0),
                  _lib.host_ptr(shading), stream_handle())
    return masks, frames


# ---- the reference's Sphere / Box scenes on the GPU (synthetic.py:21-243) ----
# SURVEY.md 8f4. analytic_silhouette, shade_frame and proposal_from_silhouette
# run as sm_100a kernels (csrc/synth.cu: fvv_synth_render, fvv_erode_cross)
# and equal the reference's numpy/scipy outputs bit for bit
# (tests/test_gpu_synth.py against tests/golden/synth.npz). The primitives
# below are parameter records for those kernels: the reference's host-side
# ray tests (ray_hits / normal_at / contains, cast_rays) have no counterpart
# here because the intersection runs on the GPU.

@dataclass
class Sphere:
    """Sphere scene primitive (fields and validation of synthetic.py:21-31)."""

    center: np.ndarray
    radius: float
    color: np.ndarray = field(default_factory=lambda: np.array([200.0, 80.0, 60.0]))

    def __post_init__(self) -> None:
        self.center = np.asarray(self.center, dtype=np.float64).reshape(3)
        self.color = np.asarray(self.color, dtype=np.float64).reshape(3)
        if self.radius <= 0:
            raise ValueError("sphere radius must be positive")

    def aabb(self):
        r = np.full(3, float(self.radius))
        return self.center - r, self.center + r

    def _record(self):
        """fvv_synth_render record: kind 0, centre, r^2, colour."""
        return [0.0, *self.center, float(self.radius) ** 2, *self.color, 0.0, 0.0]


@dataclass
class Box:
    """Axis-aligned box primitive (fields and validation of synthetic.py:58-69)."""

    lo: np.ndarray
    hi: np.ndarray
    color: np.ndarray = field(default_factory=lambda: np.array([70.0, 110.0, 200.0]))

    def __post_init__(self) -> None:
        self.lo = np.asarray(self.lo, dtype=np.float64).reshape(3)
        self.hi = np.asarray(self.hi, dtype=np.float64).reshape(3)
        self.color = np.asarray(self.color, dtype=np.float64).reshape(3)
        if np.any(self.hi <= self.lo):
            raise ValueError("box must have positive extent")

    def aabb(self):
        return np.array(self.lo), np.array(self.hi)

    def _record(self):
        """fvv_synth_render record: kind 1, lo, hi, colour."""
        return [1.0, *self.lo, *self.hi, *self.color]


def _unit(v):
    """v / |v| with |v| summed in a fixed order (OpenBLAS's ddot order on the
    reference host, independent of this host's CPU)."""
    v = [float(x) for x in np.asarray(v, dtype=np.float64).reshape(3)]
    import math

    n = math.sqrt((v[0] * v[0] + v[1] * v[1]) + v[2] * v[2])
    return np.array([v[0] / n, v[1] / n, v[2] / n])


@dataclass
class SyntheticScene:
    """synthetic.py:101-108."""

    rig: CameraRig
    objects: list
    light_dir: np.ndarray = field(default_factory=lambda: np.array([0.3, 0.5, -0.8]))

    def __post_init__(self) -> None:
        self.light_dir = _unit(self.light_dir)


def _synth_device(cam, objects, light, want_sil, want_rgb, noise=None):
    import ctypes

    import torch

    from . import _lib
    from ._device import cam_table, require_cuda, stream_handle

    dev = require_cuda()
    for o in objects:
        if not hasattr(o, "_record"):
            raise TypeError(f"unsupported object {type(o).__name__} (Sphere or Box)")
    recs = np.array([o._record() for o in objects], dtype=np.float64).reshape(-1, 10)
    d_objs = torch.from_numpy(recs).to(dev) if len(objects) else None
    h, w = cam.image_height, cam.image_width
    sil = torch.empty((h, w), dtype=torch.uint8, device=dev) if want_sil else None
    rgb = torch.empty((h, w, 3), dtype=torch.uint8, device=dev) if want_rgb else None
    d_noise = None
    if noise is not None:
        d_noise = torch.from_numpy(np.ascontiguousarray(noise, dtype=np.float64)).to(dev)
    shading = np.array([AMBIENT, 1.0 - AMBIENT, *BG_COLOR], dtype=np.float64)
    light = np.ascontiguousarray(light, dtype=np.float64)
    null = ctypes.c_void_p(0)
    _lib.call("fvv_synth_render", _lib.host_ptr(cam_table([cam])), _lib.host_ptr(light),
              _lib.host_ptr(shading), _lib.dev_ptr(d_objs) if d_objs is not None else null,
              ctypes.c_int(len(objects)), _lib.dev_ptr(d_noise) if d_noise is not None else null,
              _lib.dev_ptr(sil) if sil is not None else null,
              _lib.dev_ptr(rgb) if rgb is not None else null, stream_handle())
    return sil, rgb


def analytic_silhouette(cam, objects) -> np.ndarray:
    """Exact binary silhouette: a pixel is foreground iff its centre ray hits
    any object in front of the camera (synthetic.py:187-192), on the GPU."""
    if cam.has_distortion:
        raise ValueError("pixel_rays supports zero-distortion cameras only")  # the reference message
    sil, _ = _synth_device(cam, list(objects), np.array([0.0, 0.0, 1.0]), True, False)
    return sil.cpu().numpy().astype(bool)


def shade_frame(scene: SyntheticScene, cam, noise_sigma: float = 0.0, seed: int = 0):
    """Lambertian-shaded uint8 RGB frame, flat background, optional seeded
    Gaussian noise (synthetic.py:195-218). The noise is numpy's
    default_rng(seed + cam.id) stream, drawn on the host; the shading runs on
    the GPU."""
    if cam.has_distortion:
        raise ValueError("pixel_rays supports zero-distortion cameras only")  # the reference message
    noise = None
    if noise_sigma > 0:
        rng = np.random.default_rng(seed + cam.id)
        noise = rng.normal(0.0, noise_sigma, (cam.image_height, cam.image_width, 3))
    _, rgb = _synth_device(cam, list(scene.objects), scene.light_dir, False, True, noise)
    return rgb.cpu().numpy()


def proposal_from_silhouette(sil, erode_px: int = 3) -> np.ndarray:
    """The silhouette eroded erode_px times with the 3x3 cross, outside = 0
    (synthetic.py:221-226, scipy binary_erosion), on the GPU."""
    import ctypes

    import torch

    from . import _lib
    from ._device import require_cuda, stream_handle

    sil = np.asarray(sil, dtype=bool)
    if erode_px <= 0:
        return sil.copy()
    dev = require_cuda()
    h, w = sil.shape
    d_in = torch.from_numpy(np.ascontiguousarray(sil).view(np.uint8)).to(dev)
    tmp = torch.empty_like(d_in)
    out = torch.empty_like(d_in)
    _lib.call("fvv_erode_cross", _lib.dev_ptr(d_in), _lib.dev_ptr(tmp), _lib.dev_ptr(out),
              ctypes.c_int(w), ctypes.c_int(h), ctypes.c_int(int(erode_px)), stream_handle())
    return out.cpu().numpy().astype(bool)


def scene_silhouettes(scene: SyntheticScene) -> list:
    return [analytic_silhouette(cam, scene.objects) for cam in scene.rig]


def scene_frames(scene: SyntheticScene, noise_sigma: float = 0.0, seed: int = 0) -> list:
    return [shade_frame(scene, cam, noise_sigma, seed) for cam in scene.rig]


def validate_in_stage(objects, stage_lo, stage_hi) -> None:
    """synthetic.py:237-243."""
    stage_lo = np.asarray(stage_lo, dtype=np.float64)
    stage_hi = np.asarray(stage_hi, dtype=np.float64)
    for i, obj in enumerate(objects):
        lo, hi = obj.aabb()
        if np.any(lo < stage_lo) or np.any(hi > stage_hi):
            raise ValueError(f"object {i} extends outside the stage volume")
