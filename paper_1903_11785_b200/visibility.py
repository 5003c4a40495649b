"""Depth images and occlusion flags on the GPU (drop-in for freeview.visibility).

``rasterize`` / ``depth_image`` run fvv_rasterize (every camera of a rig in
one launch when called through ``visibility_maps``); ``classify_visibility``
runs fvv_classify. Results equal the reference's Python rasteriser bit for
bit: float64 edge functions with the top-left rule, perspective-correct
depth, lowest triangle id on exact depth ties (visibility.py:34-140).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._device import cam_table, require_cuda, stream_handle

NEAR_CLIP_MM = 1.0  # visibility.py:19


@dataclass
class RasterResult:
    depth: np.ndarray  # (H, W) float64 mm, +inf where uncovered
    tri_id: np.ndarray  # (H, W) int32, -1 where uncovered


def _plane_offsets(cams):
    sizes = [c.image_height * c.image_width for c in cams]
    off = np.zeros(len(cams), dtype=np.int64)
    off[1:] = np.cumsum(sizes)[:-1]
    return off, int(sum(sizes))


def _mesh_dev(mesh):
    """(verts, tris, nt_host_upper_bound, nt_dev or None)."""
    verts, tris = mesh.device_arrays()
    return verts, tris, int(tris.shape[0]), None


class DevicePlanes:
    """Depth (and optionally triangle-id) planes of several cameras on the GPU."""

    def __init__(self, cams, depth, tri_id, offsets):
        self.cams = list(cams)
        self.depth = depth
        self.tri_id = tri_id
        self.offsets = offsets

    def depth_of(self, c) -> torch.Tensor:
        cam = self.cams[c]
        o = int(self.offsets[c])
        return self.depth[o:o + cam.image_height * cam.image_width].view(cam.image_height,
                                                                         cam.image_width)

    def tri_id_of(self, c) -> torch.Tensor:
        cam = self.cams[c]
        o = int(self.offsets[c])
        return self.tri_id[o:o + cam.image_height * cam.image_width].view(cam.image_height,
                                                                          cam.image_width)


def raster_planes(verts, tris, cams, want_ids=False, nt_dev=None) -> DevicePlanes:
    """fvv_rasterize over ``cams``; triangles ``tris[:n]`` with n = *nt_dev
    when given (tris.shape[0] is then only an upper bound)."""
    dev = verts.device
    cams = list(cams)
    if len(cams) > _lib.FVV_MAX_CAMS:
        raise ValueError(f"{len(cams)} cameras exceed the kernel limit {_lib.FVV_MAX_CAMS}")
    tab = cam_table(cams)
    off, total = _plane_offsets(cams)
    depth = torch.empty(total, dtype=torch.float64, device=dev)
    ids = torch.empty(total, dtype=torch.int32, device=dev) if want_ids else None
    nt = int(tris.shape[0]) if tris.numel() else 0
    wsb = int(_lib.load().fvv_raster_workspace_bytes(int(verts.shape[0]), nt, len(cams)))
    ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
    _lib.call("fvv_rasterize", _lib.host_ptr(tab), ctypes.c_int(len(cams)), _lib.dev_ptr(verts),
              _lib.i64(verts.shape[0]), _lib.dev_ptr(tris), _lib.i64(nt),
              _lib.dev_ptr(nt_dev) if nt_dev is not None else ctypes.c_void_p(0),
              _lib.dev_ptr(depth), _lib.host_ptr(off),
              _lib.dev_ptr(ids) if ids is not None else ctypes.c_void_p(0), _lib.dev_ptr(ws),
              ctypes.c_size_t(wsb), stream_handle())
    planes = DevicePlanes(cams, depth, ids, off)
    planes._ws = ws
    return planes


def classify_bits(verts, tris, planes: DevicePlanes, t_v, nt_dev=None):
    """fvv_classify -> visibility bits (ncam, ceil(T/32)) int32 on the GPU."""
    dev = verts.device
    cams = planes.cams
    nt = int(tris.shape[0]) if tris.numel() else 0
    stride = max((nt + 31) // 32, 1)
    vis = torch.zeros((len(cams), stride), dtype=torch.int32, device=dev)
    if nt:
        _lib.call("fvv_classify", _lib.host_ptr(cam_table(cams)), ctypes.c_int(len(cams)),
                  _lib.dev_ptr(verts), _lib.dev_ptr(tris), _lib.i64(nt),
                  _lib.dev_ptr(nt_dev) if nt_dev is not None else ctypes.c_void_p(0),
                  _lib.dev_ptr(planes.depth), _lib.host_ptr(planes.offsets),
                  ctypes.c_double(float(t_v)), _lib.dev_ptr(vis), _lib.i64(stride),
                  stream_handle())
    return vis


def bits_to_flags(bits_row: np.ndarray, n: int) -> np.ndarray:
    return np.unpackbits(np.ascontiguousarray(bits_row).view(np.uint8),
                         bitorder="little")[:n].astype(bool)


def rasterize(mesh, cam) -> RasterResult:
    """Edge-function rasteriser with the top-left rule (visibility.py:34-98)."""
    require_cuda()
    h, w = cam.image_height, cam.image_width
    if mesh.num_triangles == 0:
        return RasterResult(np.full((h, w), np.inf), np.full((h, w), -1, dtype=np.int32))
    verts, tris, _, _ = _mesh_dev(mesh)
    planes = raster_planes(verts, tris, [cam], want_ids=True)
    return RasterResult(planes.depth_of(0).cpu().numpy(), planes.tri_id_of(0).cpu().numpy())


def depth_image(mesh, cam) -> np.ndarray:
    """Per-pixel nearest depth in mm, +inf background (visibility.py:101-103)."""
    require_cuda()
    h, w = cam.image_height, cam.image_width
    if mesh.num_triangles == 0:
        return np.full((h, w), np.inf)
    verts, tris, _, _ = _mesh_dev(mesh)
    return raster_planes(verts, tris, [cam]).depth_of(0).cpu().numpy()


def classify_visibility(mesh, cam, depth, t_v: float) -> np.ndarray:
    """Per-triangle visibility flags (visibility.py:106-129): visible iff the
    centroid is in-frustum and no more than t_v behind the cached depth."""
    if mesh.num_triangles == 0:
        return np.zeros(0, dtype=bool)
    dev = require_cuda()
    verts, tris, _, _ = _mesh_dev(mesh)
    d = torch.from_numpy(np.ascontiguousarray(depth, dtype=np.float64).reshape(-1)).to(dev)
    planes = DevicePlanes([cam], d, None, np.zeros(1, dtype=np.int64))
    bits = classify_bits(verts, tris, planes, t_v)
    return bits_to_flags(bits[0].cpu().numpy(), mesh.num_triangles)


def visibility_maps(mesh, rig, t_v: float):
    """Depth image and visibility flags for every camera (visibility.py:132-140),
    all cameras in one raster launch and one classify launch."""
    cams = list(rig)
    if mesh.num_triangles == 0:
        return ({c.id: np.full((c.image_height, c.image_width), np.inf) for c in cams},
                {c.id: np.zeros(0, dtype=bool) for c in cams})
    require_cuda()
    verts, tris, _, _ = _mesh_dev(mesh)
    planes = raster_planes(verts, tris, cams)
    bits = classify_bits(verts, tris, planes, t_v).cpu().numpy()
    depths = {c.id: planes.depth_of(i).cpu().numpy() for i, c in enumerate(cams)}
    vis = {c.id: bits_to_flags(bits[i], mesh.num_triangles) for i, c in enumerate(cams)}
    return depths, vis
