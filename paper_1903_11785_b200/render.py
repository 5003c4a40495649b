"""View-dependent rendering on the GPU (drop-in for freeview.render).

Cameras are ranked by optical-centre distance to the virtual viewpoint
(host, numpy, exactly as render.py:29-32 - it is a 16-element sort); every
triangle takes its texture from the first-ranked camera that sees it
(fvv_triangle_sources); the virtual view is rasterised (fvv_rasterize) and
each covered pixel is back-projected, re-projected through the source
camera's full distortion model and bilinearly sampled (fvv_render_view).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._device import cam_table, require_cuda, stream_handle
from .visibility import classify_bits, raster_planes  # noqa: F401  (re-exported helpers)

FALLBACK_COLOR = np.array([128, 128, 128], dtype=np.uint8)  # render.py:19

# host->device bytes of colour frames moved by the render path (bench.py reads it)
H2D_BYTES = {"frames": 0, "masks": 0}  # bytes run_sequence moved host->device
D2H_BYTES = {"results": 0}  # bytes run_sequence read back (pinned blocks)


@dataclass
class RenderedImage:
    color: np.ndarray  # (H, W, 3) uint8
    source: np.ndarray  # (H, W) int32 camera id, -1 = none
    covered: np.ndarray  # (H, W) bool


class CodedImage(RenderedImage):
    """A RenderedImage read back in compact form: colour plus one int8 code
    per pixel (-2 uncovered, -1 fallback colour, else the source camera's
    rig position, fvv_render_view_coded). ``source`` (camera ids) and
    ``covered`` are expanded from the code on first access."""

    def __init__(self, color, code, rig_ids):
        self.color = color
        self._code = code
        self._lut = np.concatenate(([-1, -1], np.asarray(rig_ids, dtype=np.int32)))
        self._source = None
        self._covered = None

    @property
    def source(self):
        if self._source is None:
            self._source = self._lut[self._code.astype(np.int64) + 2]
        return self._source

    @source.setter
    def source(self, value):
        self._source = value

    @property
    def covered(self):
        if self._covered is None:
            self._covered = self._code != -2
        return self._covered

    @covered.setter
    def covered(self, value):
        self._covered = value


def rank_cameras(virtual, rig) -> list:
    """Camera ids by ascending optical-centre distance; ties to the lower id."""
    keys = sorted((float(np.linalg.norm(c.center - virtual.center)), c.id) for c in rig)
    return [cid for _, cid in keys]


def _rank_tables(ranking, rig):
    pos = {c.id: i for i, c in enumerate(rig)}
    return (np.array([pos[i] for i in ranking], dtype=np.int32),
            np.array(ranking, dtype=np.int32))


def _vis_bits_from_dict(vis, rig, n, dev):
    stride = max((n + 31) // 32, 1)
    host = np.zeros((len(rig), stride * 4), dtype=np.uint8)
    for i, c in enumerate(rig):
        p = np.packbits(np.asarray(vis[c.id], dtype=bool)[:n], bitorder="little")
        host[i, :len(p)] = p
    return torch.from_numpy(host.view(np.int32)).to(dev), stride


def sources_device(ranking, rig, vis_bits, stride, n, nt_dev=None):
    rank_pos, rank_id = _rank_tables(ranking, rig)
    src = torch.empty(max(n, 1), dtype=torch.int32, device=vis_bits.device)
    _lib.call("fvv_triangle_sources", _lib.host_ptr(rank_pos), _lib.host_ptr(rank_id),
              ctypes.c_int(len(rank_pos)), _lib.dev_ptr(vis_bits), _lib.i64(stride), _lib.i64(n),
              _lib.dev_ptr(nt_dev) if nt_dev is not None else ctypes.c_void_p(0),
              _lib.dev_ptr(src), stream_handle())
    return src


def triangle_sources(ranking, vis, n_triangles: int) -> np.ndarray:
    """First-ranked camera id that sees each triangle; -1 if none (render.py:35-43)."""
    dev = require_cuda()
    ids = list(ranking)
    if n_triangles == 0:
        return np.zeros(0, dtype=np.int32)

    class _Cam:  # rig stand-in: positions follow the ranking order
        def __init__(self, i):
            self.id = i

    rig = [_Cam(i) for i in ids]
    bits, stride = _vis_bits_from_dict(vis, rig, n_triangles, dev)
    return sources_device(ids, rig, bits, stride, n_triangles)[:n_triangles].cpu().numpy()


def sample_bilinear(img, u, v) -> np.ndarray:
    """Host helper: bilinear sample, clamped (render.py:46-61). The render
    kernel does the same per pixel on the GPU."""
    h, w = img.shape[:2]
    u = np.clip(u, 0.0, w - 1.0)
    v = np.clip(v, 0.0, h - 1.0)
    x0 = np.floor(u).astype(np.int64)
    y0 = np.floor(v).astype(np.int64)
    x1 = np.minimum(x0 + 1, w - 1)
    y1 = np.minimum(y0 + 1, h - 1)
    fx = (u - x0)[:, None]
    fy = (v - y0)[:, None]
    f = img.astype(np.float64)
    top = f[y0, x0] * (1 - fx) + f[y0, x1] * fx
    bot = f[y1, x0] * (1 - fx) + f[y1, x1] * fx
    return top * (1 - fy) + bot * fy


def frames_device(rig, frames, dev):
    """(H,W,3) uint8 frames of every rig camera, concatenated on the GPU."""
    sizes = [c.image_height * c.image_width * 3 for c in rig]
    off = np.zeros(len(sizes), dtype=np.int64)
    off[1:] = np.cumsum(sizes)[:-1]
    buf = torch.empty(max(int(sum(sizes)), 1), dtype=torch.uint8, device=dev)
    for c, o, sz in zip(rig, off, sizes):
        f = frames[c.id]
        t = f if isinstance(f, torch.Tensor) else torch.from_numpy(
            np.ascontiguousarray(np.asarray(f, dtype=np.uint8)))
        buf[int(o):int(o) + sz].copy_(t.reshape(-1), non_blocking=True)
    return buf, off


def _frame_tensor(f):
    if isinstance(f, torch.Tensor):
        return f
    return torch.from_numpy(np.ascontiguousarray(np.asarray(f, dtype=np.uint8)))


def render_device(verts, tris, nt, rig, frames, vis_bits, stride, virtual,
                  fallback_color=FALLBACK_COLOR, nt_dev=None, frame_buf=None, prefetched=None):
    """Device-side render_view -> (color, source, covered, counts) GPU tensors.

    Colour frames come either as ``frame_buf = (device buffer, offsets)``
    holding every rig camera, or as the reference's ``frames`` dict of host
    (H, W, 3) arrays; then only the cameras that actually source a pixel are
    copied to the GPU (after fvv_render_count), reusing ``prefetched``
    {rig position: device tensor} when given."""
    dev = verts.device
    rig = list(rig)
    h, w = virtual.image_height, virtual.image_width
    planes = raster_planes(verts, tris[:max(nt, 0)] if nt_dev is None else tris, [virtual],
                           want_ids=True, nt_dev=nt_dev)
    ranking = rank_cameras(virtual, rig)
    src = sources_device(ranking, rig, vis_bits, stride, max(nt, 1), nt_dev)
    tab = cam_table(rig)
    vtab = cam_table([virtual])
    counts = torch.empty(1 + len(rig), dtype=torch.int64, device=dev)
    _lib.call("fvv_render_count", _lib.host_ptr(tab), ctypes.c_int(len(rig)),
              _lib.host_ptr(vtab), _lib.dev_ptr(planes.tri_id), _lib.dev_ptr(src),
              _lib.dev_ptr(counts), stream_handle())
    if frame_buf is not None:
        buf, off = frame_buf
    else:
        used = np.flatnonzero(counts[1:].cpu().numpy() > 0)  # sync: which frames are read
        prefetched = prefetched or {}
        sizes = [rig[c].image_height * rig[c].image_width * 3 for c in used]
        off = np.zeros(len(rig), dtype=np.int64)
        buf = torch.empty(max(int(sum(sizes)), 1), dtype=torch.uint8, device=dev)
        o = 0
        for c, sz in zip(used, sizes):
            off[c] = o
            t = prefetched.get(int(c))
            if t is None:
                t = _frame_tensor(frames[rig[c].id])
                H2D_BYTES["frames"] += sz
            buf[o:o + sz].copy_(t.reshape(-1), non_blocking=True)
            o += sz
    color = torch.empty((h, w, 3), dtype=torch.uint8, device=dev)
    source = torch.empty((h, w), dtype=torch.int32, device=dev)
    covered = torch.empty((h, w), dtype=torch.uint8, device=dev)
    fb = np.ascontiguousarray(np.asarray(fallback_color, dtype=np.uint8).reshape(3))
    _lib.call("fvv_render_view", _lib.host_ptr(tab), ctypes.c_int(len(rig)),
              _lib.dev_ptr(buf), _lib.host_ptr(off), _lib.host_ptr(vtab),
              _lib.dev_ptr(planes.depth), _lib.dev_ptr(planes.tri_id), _lib.dev_ptr(src),
              _lib.host_ptr(fb), _lib.dev_ptr(color), _lib.dev_ptr(source),
              _lib.dev_ptr(covered), _lib.dev_ptr(counts), stream_handle())
    return color, source, covered, counts


def render_view(mesh, rig, frames: dict, vis: dict, virtual, fallback_color=FALLBACK_COLOR):
    """Rasterise the mesh from ``virtual`` and texture every pixel from the
    best-ranked camera that sees its triangle (render.py:64-113)."""
    for cam in rig:
        if cam.id not in frames:
            raise ValueError(f"missing frame for camera {cam.id}")
        if cam.id not in vis:
            raise ValueError(f"missing visibility for camera {cam.id}")
    dev = require_cuda()
    h, w = virtual.image_height, virtual.image_width
    rig = list(rig)
    if mesh.num_triangles == 0:
        return RenderedImage(np.zeros((h, w, 3), np.uint8), np.full((h, w), -1, np.int32),
                             np.zeros((h, w), bool))
    verts, tris = mesh.device_arrays()
    n = mesh.num_triangles
    dbits = getattr(vis, "_device_bits", None)
    if dbits is not None and getattr(vis, "_n", -1) == n and list(vis) == [c.id for c in rig]:
        bits, stride = dbits, int(dbits.shape[1])  # run_frame's bits, still on the GPU
    else:
        bits, stride = _vis_bits_from_dict(vis, rig, n, dev)
    color, source, covered, counts = render_device(verts, tris, n, rig, frames, bits, stride,
                                                   virtual, fallback_color)
    cov = covered.cpu().numpy().astype(bool)
    if virtual.has_distortion and cov.any():
        raise ValueError("back_project supports zero-distortion cameras only")
    return RenderedImage(color.cpu().numpy(), source.cpu().numpy(), cov)


def source_map_image(rendered: RenderedImage, rig) -> np.ndarray:
    """Host helper: false-colour view of the per-pixel source camera (render.py:116-131)."""
    palette = np.array([[230, 60, 60], [60, 180, 75], [65, 105, 225], [240, 180, 40],
                        [170, 70, 200], [70, 200, 200], [245, 130, 48], [140, 220, 90],
                        [200, 100, 160], [100, 140, 240], [180, 180, 60], [90, 90, 90]],
                       dtype=np.uint8)
    out = np.zeros((*rendered.source.shape, 3), dtype=np.uint8)
    for pos, cid in enumerate(sorted(c.id for c in rig)):
        out[rendered.source == cid] = palette[pos % len(palette)]
    out[rendered.covered & (rendered.source == -1)] = [255, 255, 255]
    return out
