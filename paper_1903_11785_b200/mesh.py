"""Exact-isovalue marching cubes on the GPU (drop-in for freeview.mesh).

``polygonize`` runs fvv_mesh_prepare / fvv_mesh_emit (include/fvv.h): edge
isovalues by Bresenham walks against the bit-packed silhouettes, vertices,
slot-major triangles with reversed winding and the degenerate-area filter,
all in the reference's float64 order and output order (mesh.py:275-374).
The pipeline calls ``polygonize_grids`` to mesh every ROI grid of a frame in
one batch. ``bresenham_line``/``bresenham_batch`` are the reference's small
host helpers (the kernels walk lines themselves).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._device import DeviceSilhouettes, cam_table, grid_table, require_cuda, stream_handle

DEGENERATE_AREA_MM2 = 1e-9  # mesh.py:22

# Bourke cube geometry (mesh.py:25-38): corners, edge base offsets, edge axes
CORNER_OFFSETS = np.array([(0, 0, 0), (1, 0, 0), (1, 1, 0), (0, 1, 0),
                           (0, 0, 1), (1, 0, 1), (1, 1, 1), (0, 1, 1)], dtype=np.int64)
EDGE_BASE = np.array([(0, 0, 0), (1, 0, 0), (0, 1, 0), (0, 0, 0), (0, 0, 1), (1, 0, 1),
                      (0, 1, 1), (0, 0, 1), (0, 0, 0), (1, 0, 0), (1, 1, 0), (0, 1, 0)],
                     dtype=np.int64)
EDGE_AXIS = np.array([0, 1, 0, 1, 0, 1, 0, 1, 2, 2, 2, 2], dtype=np.int64)


@dataclass
class EdgeIntersection:
    """mesh.py:41-50."""

    p_on: np.ndarray
    p_off: np.ndarray
    lam: float
    contributing_camera: int = -1

    @property
    def point(self) -> np.ndarray:
        return self.p_on + self.lam * (self.p_off - self.p_on)


@dataclass
class IsovalueStats:
    """mesh.py:225-228."""

    fallback_edges: int = 0
    inconsistent_starts: int = 0


class TriangleMesh:
    """Indexed triangle mesh (mesh.py:53-105): vertices float64 (V,3),
    triangles int32 (T,3), object_ids int32 (T,).

    Meshes produced on the GPU keep device copies for the visibility and
    render kernels and load their host arrays on first access."""

    def __init__(self, vertices, triangles, object_ids=None):
        self._set_host(vertices, triangles, object_ids)
        self._loader = None
        self._dev = None

    def _set_host(self, vertices, triangles, object_ids):
        v = np.asarray(vertices, dtype=np.float64).reshape(-1, 3)
        t = np.asarray(triangles, dtype=np.int32).reshape(-1, 3)
        o = np.zeros(len(t), dtype=np.int32) if object_ids is None else \
            np.asarray(object_ids, dtype=np.int32).reshape(-1)
        if len(o) != len(t):
            raise ValueError("object_ids length must match triangle count")
        if len(t) and t.max(initial=-1) >= len(v):
            raise ValueError("triangle index out of range")
        self._v, self._t, self._o = v, t, o
        self._nt = len(t)

    @classmethod
    def _trusted(cls, vertices, triangles, object_ids, dev=None):
        """Wrap kernel outputs without re-validating them (they come from
        the mesh kernels, whose indices are in range by construction).
        ``object_ids`` may be a callable producing them on first access."""
        m = cls.__new__(cls)
        m._v, m._t, m._o = vertices, triangles, object_ids
        m._nt = len(triangles)
        m._loader = None
        m._dev = dev
        return m

    @classmethod
    def _lazy(cls, num_triangles, loader, dev=None):
        m = cls.__new__(cls)
        m._v = m._t = m._o = None
        m._nt = int(num_triangles)
        m._loader = loader
        m._dev = dev
        return m

    def _load(self):
        if self._v is None:
            v, t, o = self._loader()
            self._set_host(v, t, o)

    @property
    def vertices(self) -> np.ndarray:
        self._load()
        return self._v

    @vertices.setter
    def vertices(self, value):
        self._load()
        self._set_host(value, self._t, self.object_ids)
        self._dev = None

    @property
    def triangles(self) -> np.ndarray:
        self._load()
        return self._t

    @triangles.setter
    def triangles(self, value):
        self._load()
        self._set_host(self._v, value, None)
        self._dev = None

    @property
    def object_ids(self) -> np.ndarray:
        self._load()
        if callable(self._o):  # _trusted with deferred ids
            self._o = self._o()
        return self._o

    @object_ids.setter
    def object_ids(self, value):
        self._load()
        self._set_host(self._v, self._t, value)

    @property
    def num_triangles(self) -> int:
        return self._nt

    def device_arrays(self, device=None):
        """(vertices float64 (V,3), triangles int32 (T,3)) on the GPU; the
        triangle indices address the returned vertex array."""
        if self._dev is None:
            dev = device or require_cuda()
            self._dev = (torch.from_numpy(np.ascontiguousarray(self.vertices)).to(dev),
                         torch.from_numpy(np.ascontiguousarray(self.triangles)).to(dev))
        return self._dev

    def triangle_vertices(self) -> np.ndarray:
        return self.vertices[self.triangles]

    def areas(self) -> np.ndarray:
        """Host helper (mesh.py:78-82)."""
        tv = self.triangle_vertices()
        return 0.5 * np.linalg.norm(np.cross(tv[:, 1] - tv[:, 0], tv[:, 2] - tv[:, 0]), axis=1)

    def centroids(self) -> np.ndarray:
        """Host helper (mesh.py:84-85)."""
        return self.triangle_vertices().mean(axis=1)

    @staticmethod
    def empty() -> "TriangleMesh":
        return TriangleMesh(np.zeros((0, 3)), np.zeros((0, 3), dtype=np.int32))

    @staticmethod
    def concatenate(meshes) -> "TriangleMesh":
        """Offset and join meshes, dropping those without triangles (mesh.py:92-105)."""
        meshes = [m for m in meshes if m.num_triangles]
        if not meshes:
            return TriangleMesh.empty()
        verts, tris, oids, base = [], [], [], 0
        for m in meshes:
            verts.append(m.vertices)
            tris.append(m.triangles + base)
            oids.append(m.object_ids)
            base += len(m.vertices)
        return TriangleMesh(np.concatenate(verts), np.concatenate(tris), np.concatenate(oids))

    def __repr__(self) -> str:
        return f"TriangleMesh(triangles={self._nt})"


# ---------------------------------------------------------------- helpers
def bresenham_line(x0: int, y0: int, x1: int, y1: int) -> list:
    """Host helper: integer line, endpoints inclusive (mesh.py:108-128)."""
    dx, dy = abs(x1 - x0), -abs(y1 - y0)
    sx, sy = (1 if x1 >= x0 else -1), (1 if y1 >= y0 else -1)
    err, x, y = dx + dy, x0, y0
    out = []
    while True:
        out.append((x, y))
        if x == x1 and y == y1:
            return out
        e2 = 2 * err
        if e2 >= dy:
            err += dy
            x += sx
        if e2 <= dx:
            err += dx
            y += sy


def bresenham_batch(a, b):
    """Host helper: closed-form Bresenham over many segments
    (mesh.py:131-162) -> (pixels (N, L, 2), valid (N, L))."""
    a = np.asarray(a, dtype=np.int64).reshape(-1, 2)
    b = np.asarray(b, dtype=np.int64).reshape(-1, 2)
    d = np.abs(b - a)
    s = np.where(b >= a, 1, -1)
    major = d.max(axis=1)
    lmax = int((major + 1).max(initial=1))
    t = np.arange(lmax, dtype=np.int64)[None, :]
    valid = t < (major + 1)[:, None]
    tc = np.minimum(t, major[:, None])
    xmaj = d[:, 0] >= d[:, 1]
    dmaj = np.maximum(major, 1)[:, None]
    dmin = np.where(xmaj, d[:, 1], d[:, 0])[:, None]
    smin = (2 * tc * dmin + dmaj) // (2 * dmaj)
    px = np.empty((len(a), lmax, 2), dtype=np.int64)
    px[:, :, 0] = a[:, :1] + s[:, :1] * np.where(xmaj[:, None], tc, smin)
    px[:, :, 1] = a[:, 1:2] + s[:, 1:2] * np.where(xmaj[:, None], smin, tc)
    return px, valid


def _by_id(dsils: DeviceSilhouettes, rig):
    order = sorted(range(len(rig)), key=lambda i: rig[i].id)
    return (np.ascontiguousarray(dsils.cams[order]),
            np.ascontiguousarray(dsils.word_off[order]), len(order))


def _edge_isovalues_batch(rig, sils, p_on, p_off):
    """Per-edge min-over-cameras isovalues on the GPU (mesh.py:231-272)
    -> (lam (E,), camera id (E,), IsovalueStats)."""
    dev = require_cuda()
    dsils = sils if isinstance(sils, DeviceSilhouettes) else DeviceSilhouettes(rig, sils)
    p_on = np.ascontiguousarray(np.asarray(p_on, dtype=np.float64).reshape(-1, 3))
    p_off = np.ascontiguousarray(np.asarray(p_off, dtype=np.float64).reshape(-1, 3))
    n = len(p_on)
    d_on, d_off = torch.from_numpy(p_on).to(dev), torch.from_numpy(p_off).to(dev)
    lam = torch.empty(max(n, 1), dtype=torch.float64, device=dev)
    cam = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    stats = torch.zeros(2, dtype=torch.int64, device=dev)
    cams, offs, ncam = _by_id(dsils, rig)
    _lib.call("fvv_edge_isovalues", _lib.host_ptr(cams), ctypes.c_int(ncam),
              _lib.dev_ptr(dsils.bits), _lib.host_ptr(offs), _lib.dev_ptr(d_on),
              _lib.dev_ptr(d_off), _lib.i64(n), _lib.dev_ptr(lam), _lib.dev_ptr(cam),
              _lib.dev_ptr(stats), stream_handle())
    st = stats.cpu().tolist()
    return (lam[:n].cpu().numpy(), cam[:n].cpu().numpy().astype(np.int64),
            IsovalueStats(fallback_edges=int(st[0]), inconsistent_starts=int(st[1])))


def edge_isovalue_cam(cam, sil, p_on, p_off):
    """Single-camera isovalue (mesh.py:170-198) -> (lam, start_on_bg)."""
    from .camera import CameraRig, project

    p_on = np.asarray(p_on, dtype=np.float64)
    p_off = np.asarray(p_off, dtype=np.float64)
    if not (project(cam, p_on)[2] and project(cam, p_off)[2]):
        raise ValueError("both endpoints must be in-frustum")
    lam, _, st = _edge_isovalues_batch(CameraRig([cam]), [sil], p_on[None], p_off[None])
    return float(lam[0]), st.inconsistent_starts > 0


def edge_isovalue(rig, sils, p_on, p_off) -> EdgeIntersection:
    """Minimum isovalue over the cameras seeing both endpoints; ties to the
    lowest id; 0.5 and camera -1 when none qualifies (mesh.py:201-222)."""
    p_on = np.asarray(p_on, dtype=np.float64)
    p_off = np.asarray(p_off, dtype=np.float64)
    lam, cam, _ = _edge_isovalues_batch(rig, sils, p_on[None], p_off[None])
    return EdgeIntersection(p_on, p_off, float(lam[0]), int(cam[0]))


# ------------------------------------------------------------ polygonize
_INFO_VBASE, _INFO_V, _INFO_SBASE, _INFO_S, _INFO_TBASE, _INFO_T, _INFO_FB, _INFO_INC = range(8)


def _shared_occ(grids, dev):
    """One device buffer holding every grid's occupancy words + word offsets
    (grids carved in one batch already share one buffer)."""
    bits = [g.device_bits(dev) for g in grids]
    st0 = bits[0].untyped_storage()
    if all(b.untyped_storage().data_ptr() == st0.data_ptr() for b in bits):
        base = min(b.data_ptr() for b in bits)
        buf = torch.empty(0, dtype=torch.int32, device=dev).set_(
            st0, (base - st0.data_ptr()) // 4,
            ((max(b.data_ptr() + 4 * b.numel() for b in bits) - base) // 4,))
        return buf, np.array([(b.data_ptr() - base) // 4 for b in bits], dtype=np.int64)
    offs = np.zeros(len(bits), dtype=np.int64)
    offs[1:] = np.cumsum([b.numel() for b in bits])[:-1]
    return torch.cat(bits), offs


class MeshBatch:
    """Device result of polygonizing several grids in one launch sequence."""

    def __init__(self, grids, verts, tris, ws, tab, object_ids, exact):
        self.grids = grids
        self.verts = verts      # float64 (V, 3) on the GPU
        self.tris = tris        # int32 (<=5S, 3) on the GPU, indices into verts
        self._ws = ws
        self._tab = tab
        self.object_ids = list(object_ids)
        self.exact = exact
        dev = verts.device
        self._totals = torch.zeros(3, dtype=torch.int64, device=dev)
        self._info = torch.zeros((len(grids), 8), dtype=torch.int64, device=dev)
        _lib.call("fvv_mesh_counts", _lib.host_ptr(tab), ctypes.c_int(len(grids)),
                  _lib.dev_ptr(ws), _lib.dev_ptr(self._totals), _lib.dev_ptr(self._info),
                  stream_handle())
        self._host = None

    @property
    def num_triangles_dev(self):
        """Device scalar (int64) with the total triangle count."""
        return self._totals[2:3]

    def host_info(self):
        if self._host is None:
            both = torch.cat([self._totals, self._info.reshape(-1)]).cpu().numpy()
            self._host = (both[:3].copy(), both[3:].reshape(len(self.grids), 8).copy())
        return self._host

    def stats(self, g) -> IsovalueStats:
        info = self.host_info()[1][g]
        if not self.exact:
            return IsovalueStats()
        return IsovalueStats(int(info[_INFO_FB]), int(info[_INFO_INC]))

    def host_arrays(self):
        """All vertices (V,3) and triangles (T,3) (indices into the batch's
        vertex array) copied to the host in two transfers, cached."""
        if getattr(self, "_host_arrays", None) is None:
            totals, _ = self.host_info()
            nt = int(totals[2])
            v = torch.empty(self.verts.shape, dtype=torch.float64, pin_memory=True)
            t = torch.empty((nt, 3), dtype=torch.int32, pin_memory=True)
            v.copy_(self.verts, non_blocking=True)
            t.copy_(self.tris[:nt], non_blocking=True)
            torch.cuda.current_stream().synchronize()
            self._host_arrays = (v.numpy(), t.numpy())
        return self._host_arrays

    def mesh(self, g) -> TriangleMesh:
        info = self.host_info()[1][g]
        vb, nv, tb, nt = (int(info[k]) for k in (_INFO_VBASE, _INFO_V, _INFO_TBASE, _INFO_T))
        oid = self.object_ids[g]
        if nv == 0:
            return TriangleMesh.empty()

        def load():
            v, t = self.host_arrays()
            return v[vb:vb + nv], t[tb:tb + nt] - np.int32(vb), np.full(nt, oid, dtype=np.int32)

        return TriangleMesh._lazy(nt, load)

    def meshes(self):
        return [self.mesh(g) for g in range(len(self.grids))]

    def merged(self) -> TriangleMesh:
        """TriangleMesh.concatenate(meshes) (mesh.py:92-105) with device arrays
        attached; the device triangles index the batch's full vertex array
        (same positions, same triangle order as the concatenation)."""
        totals, info = self.host_info()
        nt = int(totals[2])
        meshes = self.meshes()

        def load():
            # grids with vertices but no surviving triangle are dropped by
            # concatenate; when there are none, the batch arrays ARE the merge
            if np.all((info[:, _INFO_V] == 0) | (info[:, _INFO_T] > 0)):
                v, t = self.host_arrays()
                oids = np.repeat(np.asarray(self.object_ids, dtype=np.int32), info[:, _INFO_T])
                return v, t, oids
            m = TriangleMesh.concatenate(meshes)
            return m.vertices, m.triangles, m.object_ids

        return TriangleMesh._lazy(nt, load, dev=(self.verts, self.tris[:nt]))


def polygonize_grids(grids, rig=None, sils=None, mode="exact", fixed_isovalue=0.5,
                     object_ids=None) -> MeshBatch:
    """Polygonize every grid in one batched launch sequence (one host sync
    to size the outputs)."""
    if mode not in ("exact", "fixed"):
        raise ValueError(f"unknown mode {mode!r}")
    if mode == "exact" and (rig is None or sils is None):
        raise ValueError("exact mode requires a rig and silhouettes")
    grids = list(grids)
    if len(grids) > _lib.FVV_MAX_GRIDS:
        raise ValueError(f"{len(grids)} grids exceed the batch limit {_lib.FVV_MAX_GRIDS}")
    dev = require_cuda()
    object_ids = list(object_ids) if object_ids is not None else [0] * len(grids)
    exact = mode == "exact"
    if exact:
        dsils = sils if isinstance(sils, DeviceSilhouettes) else DeviceSilhouettes(rig, sils)
        cams, offs, ncam = _by_id(dsils, rig)
        sil_ptr = _lib.dev_ptr(dsils.bits)
    else:
        cams = np.zeros(1, dtype=_lib.CAM_DTYPE)
        offs = np.zeros(1, dtype=np.int64)
        ncam, sil_ptr = 0, ctypes.c_void_p(0)
    occ, word_off = _shared_occ(grids, dev)
    tab = grid_table([g.spec for g in grids])
    ng = ctypes.c_int(len(grids))
    nbytes = int(_lib.load().fvv_mesh_workspace_bytes(_lib.host_ptr(tab), ng))
    ws = torch.empty(max(nbytes, 1), dtype=torch.uint8, device=dev)
    _lib.call("fvv_mesh_prepare", _lib.host_ptr(tab), ng, _lib.dev_ptr(occ),
              _lib.host_ptr(word_off), _lib.dev_ptr(ws), ctypes.c_size_t(nbytes), stream_handle())
    totals = torch.zeros(3, dtype=torch.int64, device=dev)
    _lib.call("fvv_mesh_counts", _lib.host_ptr(tab), ng, _lib.dev_ptr(ws), _lib.dev_ptr(totals),
              ctypes.c_void_p(0), stream_handle())
    nv, ns = (int(x) for x in totals[:2].cpu().tolist())  # the one sync: size the outputs
    sbytes = int(_lib.load().fvv_mesh_emit_scratch_bytes(nv, ns))
    scratch = torch.empty(max(sbytes, 1), dtype=torch.uint8, device=dev)
    verts = torch.empty((max(nv, 1), 3), dtype=torch.float64, device=dev)
    tris = torch.empty((max(5 * ns, 1), 3), dtype=torch.int32, device=dev)
    _lib.call("fvv_mesh_emit", _lib.host_ptr(cams), ctypes.c_int(ncam), sil_ptr,
              _lib.host_ptr(offs), _lib.host_ptr(tab), ng, _lib.dev_ptr(occ),
              _lib.host_ptr(word_off), ctypes.c_int(int(exact)), ctypes.c_double(fixed_isovalue),
              _lib.dev_ptr(ws), ctypes.c_size_t(nbytes), _lib.i64(nv), _lib.i64(ns),
              _lib.dev_ptr(scratch), ctypes.c_size_t(sbytes), _lib.dev_ptr(verts),
              _lib.dev_ptr(tris), stream_handle())
    batch = MeshBatch(grids, verts[:nv], tris, ws, tab, object_ids, exact)
    batch._scratch = scratch
    return batch


def polygonize(grid, rig=None, sils=None, mode: str = "exact", fixed_isovalue: float = 0.5,
               object_id: int = 0):
    """Marching cubes over occupancy with silhouette-exact ("exact") or
    constant ("fixed") edge isovalues (mesh.py:275-374) on the GPU.
    Returns (TriangleMesh, IsovalueStats)."""
    batch = polygonize_grids([grid], rig, sils, mode, fixed_isovalue, [object_id])
    return batch.mesh(0), batch.stats(0)
