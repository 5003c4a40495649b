"""CPU ORACLE — test infrastructure, never the product path.

Python face of ``oracle/oracle.c`` (a C restatement of the reference
``freeview`` hot path) plus the few numpy host steps the reference runs
outside its compute kernels (filter/ROI bookkeeping, camera ranking,
per-triangle sources, mesh concatenation), each restated from the
reference file:line it follows.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU
baseline leg may import this package. Pinned against the reference's own
outputs in ``tests/golden/`` (see scripts/make_golden.py).

Cameras and rigs are duck-typed: anything with the reference
``CameraModel`` attributes (id, image_width, image_height, fx, fy, cx, cy,
skew, dist, rotation, translation) works, so the same oracle checks the
reference objects and this repo's objects.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "liboracle.so")
_lib = None

CAM_DTYPE = np.dtype(
    [
        ("R", "<f8", (9,)),
        ("t", "<f8", (3,)),
        ("fx", "<f8"), ("fy", "<f8"), ("cx", "<f8"), ("cy", "<f8"), ("skew", "<f8"),
        ("k1", "<f8"), ("k2", "<f8"), ("p1", "<f8"), ("p2", "<f8"), ("k3", "<f8"),
        ("width", "<i4"), ("height", "<i4"), ("id", "<i4"), ("has_distortion", "<i4"),
    ]
)
assert CAM_DTYPE.itemsize == 192

CARVE_CHUNK = 1 << 20  # hull.py:20
DEFAULT_VOXEL_BUDGET = 400_000_000  # voxels.py:15
FALLBACK_COLOR = np.array([128, 128, 128], dtype=np.uint8)  # render.py:19


class _Mesh(ctypes.Structure):
    _fields_ = [
        ("nv", ctypes.c_int64), ("nt", ctypes.c_int64),
        ("verts", ctypes.POINTER(ctypes.c_double)), ("tris", ctypes.POINTER(ctypes.c_int32)),
        ("fallback_edges", ctypes.c_int64), ("inconsistent_starts", ctypes.c_int64),
    ]


def build() -> str:
    """Compile liboracle.so (gcc; no GPU needed)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(
            os.path.join(_HERE, "oracle.c")
        ):
            build()
        _lib = ctypes.CDLL(_LIB_PATH)
        _lib.or_label.restype = ctypes.c_int64
        _lib.or_polygonize.restype = ctypes.c_int
    return _lib


def _p(a):
    p = ctypes.c_void_p(a.ctypes.data)
    p._keep = a  # inline temporaries must outlive the call
    return p


def cam_struct(cams) -> np.ndarray:
    cams = list(cams)
    out = np.zeros(len(cams), dtype=CAM_DTYPE)
    for i, c in enumerate(cams):
        dist = np.asarray(c.dist, dtype=np.float64).reshape(5)
        out[i]["R"] = np.asarray(c.rotation, dtype=np.float64).reshape(9)
        out[i]["t"] = np.asarray(c.translation, dtype=np.float64).reshape(3)
        for k in ("fx", "fy", "cx", "cy", "skew"):
            out[i][k] = float(getattr(c, k))
        out[i]["k1"], out[i]["k2"], out[i]["p1"], out[i]["p2"], out[i]["k3"] = dist
        out[i]["width"], out[i]["height"] = int(c.image_width), int(c.image_height)
        out[i]["id"] = int(c.id)
        out[i]["has_distortion"] = int(bool(np.any(dist != 0.0)))
    return out


def _pack_images(images, channels=1):
    """Concatenate per-camera arrays into one uint8 buffer + offsets."""
    flat = [np.ascontiguousarray(np.asarray(im, dtype=np.uint8 if channels == 3 else bool)).view(np.uint8).ravel()
            for im in images]
    off = np.zeros(len(flat), dtype=np.int64)
    if flat:
        off[1:] = np.cumsum([f.size for f in flat])[:-1]
    buf = np.concatenate(flat) if flat else np.zeros(1, dtype=np.uint8)
    return np.ascontiguousarray(buf), off


def check_sils(rig, sils):
    """hull.py:63-75 (_check_sils), same messages."""
    if len(sils) != len(rig):
        raise ValueError(f"{len(sils)} silhouettes for {len(rig)} cameras")
    out = []
    for cam, sil in zip(rig, sils):
        s = np.asarray(sil, dtype=bool)
        if s.shape != (cam.image_height, cam.image_width):
            raise ValueError(
                f"camera {cam.id}: silhouette shape {s.shape} != "
                f"({cam.image_height}, {cam.image_width})"
            )
        out.append(s)
    return out


# ------------------------------------------------------------------ camera
def project(cam, pts, use_distortion=True):
    """camera.py:164-201 for an (N, 3) array -> (pixel (N,2), z (N,), in (N,))."""
    pts = np.ascontiguousarray(np.atleast_2d(np.asarray(pts, dtype=np.float64)))
    n = len(pts)
    px = np.empty((n, 2))
    z = np.empty(n)
    inf = np.empty(n, dtype=np.uint8)
    cs = cam_struct([cam])
    lib().or_project(_p(cs), _p(pts), ctypes.c_int64(n), ctypes.c_int(int(use_distortion)),
                     _p(px), _p(z), _p(inf))
    return px, z, inf.astype(bool)


# ------------------------------------------------------------------ voxels
def grid_from_aabb(lo, hi, spacing, budget=DEFAULT_VOXEL_BUDGET):
    """voxels.py:62-71 (GridSpec.from_aabb) -> (origin, spacing, dims)."""
    lo = np.asarray(lo, dtype=np.float64)
    hi = np.asarray(hi, dtype=np.float64)
    if np.any(hi <= lo):
        raise ValueError("AABB must have positive extent on every axis")
    dims = np.ceil((hi - lo) / spacing - 1e-9).astype(int)
    dims = np.maximum(dims, 1)
    dims = tuple(int(d) for d in dims)
    if dims[0] * dims[1] * dims[2] > budget:
        raise ValueError(f"grid of {dims[0] * dims[1] * dims[2]} voxels exceeds budget {budget}")
    return lo.reshape(3), float(spacing), dims


# -------------------------------------------------------------------- hull
def carve(rig, sils, origin, spacing, dims, min_views=1):
    """hull.py:95-119 -> flat bool occupancy (index i + nx*(j + ny*k))."""
    sils = check_sils(rig, sils)
    cs = cam_struct(rig)
    buf, off = _pack_images(sils)
    origin = np.ascontiguousarray(np.asarray(origin, dtype=np.float64).reshape(3))
    d = np.asarray(dims, dtype=np.int64)
    occ = np.zeros(int(d.prod()), dtype=np.uint8)
    lib().or_carve(_p(cs), ctypes.c_int(len(cs)), _p(buf), _p(off), _p(origin),
                   ctypes.c_double(spacing), _p(d), ctypes.c_int(int(min_views)), _p(occ))
    return occ.astype(bool)


@dataclass
class Component:  # hull.py:23-28
    id: int
    voxel_count: int
    bbox_min: tuple
    bbox_max: tuple


def label(occ, dims):
    """hull.py:218-254 semantics by BFS -> (labels int32, [Component])."""
    occ = np.ascontiguousarray(np.asarray(occ, dtype=bool)).view(np.uint8)
    d = np.asarray(dims, dtype=np.int64)
    labels = np.zeros(int(d.prod()), dtype=np.int32)
    n_on = int(occ.sum())
    comps = np.zeros((max(n_on, 1), 7), dtype=np.int64)
    n = lib().or_label(_p(occ), _p(d), _p(labels), _p(comps))
    out = [Component(c + 1, int(comps[c, 0]), tuple(int(v) for v in comps[c, 1:4]),
                     tuple(int(v) for v in comps[c, 4:7])) for c in range(n)]
    return labels, out


def filter_noise(labels, comps, t_small, t_large=np.inf):
    """hull.py:257-269: keep t_small <= count <= t_large, ids unchanged."""
    keeps = lambda c: t_small <= c.voxel_count <= t_large  # noqa: E731  (hull.py:46-47)
    keep_ids = np.array([c.id for c in comps if keeps(c)], dtype=np.int32)
    keep_set = np.zeros(len(comps) + 1, dtype=bool)
    keep_set[keep_ids] = True
    new_labels = np.where(keep_set[labels], labels, 0)
    return new_labels > 0, new_labels, [c for c in comps if keeps(c)]


def extract_rois(comps, origin, spacing, dims, margin):
    """hull.py:272-284 -> [(lo, hi, component_id)]."""
    origin = np.asarray(origin, dtype=np.float64)
    stage_hi = origin + spacing * np.asarray(dims, dtype=np.float64)  # voxels.py:42-44
    rois = []
    for c in comps:
        lo = origin + spacing * np.asarray(c.bbox_min, dtype=np.float64) - margin
        hi = origin + spacing * (np.asarray(c.bbox_max, dtype=np.float64) + 1.0) + margin
        lo = np.maximum(lo, origin)
        hi = np.minimum(hi, stage_hi)
        if np.any(lo >= hi):
            raise ValueError("ROI must have positive extent")
        rois.append((lo, hi, c.id))
    return rois


# -------------------------------------------------------------------- mesh
def polygonize(occ, origin, spacing, dims, rig=None, sils=None, mode="exact",
               fixed_isovalue=0.5, object_id=0):
    """mesh.py:275-374 -> (verts (V,3) f64, tris (T,3) i32, oids (T,), stats dict)."""
    if mode not in ("exact", "fixed"):
        raise ValueError(f"unknown mode {mode!r}")
    if mode == "exact" and (rig is None or sils is None):
        raise ValueError("exact mode requires a rig and silhouettes")
    occ = np.ascontiguousarray(np.asarray(occ, dtype=bool)).view(np.uint8)
    origin = np.ascontiguousarray(np.asarray(origin, dtype=np.float64).reshape(3))
    d = np.asarray(dims, dtype=np.int64)
    if mode == "exact":
        cs = cam_struct(rig)
        buf, off = _pack_images(check_sils(rig, sils))
        ncam = len(cs)
    else:
        cs = np.zeros(1, dtype=CAM_DTYPE)
        buf, off = np.zeros(1, dtype=np.uint8), np.zeros(1, dtype=np.int64)
        ncam = 0
    m = _Mesh()
    rc = lib().or_polygonize(_p(occ), _p(origin), ctypes.c_double(spacing), _p(d), _p(cs),
                             ctypes.c_int(ncam), _p(buf), _p(off), ctypes.c_int(mode == "exact"),
                             ctypes.c_double(fixed_isovalue), ctypes.byref(m))
    if rc != 0:
        raise MemoryError("oracle polygonize allocation failed")
    try:
        nv, nt = m.nv, m.nt
        stats = {"fallback_edges": int(m.fallback_edges),
                 "inconsistent_starts": int(m.inconsistent_starts)}
        if nt == 0:
            # mesh.py:298-310,361-362: no surface cells -> TriangleMesh.empty();
            # all-degenerate keeps the vertices with zero triangles
            verts = (np.ctypeslib.as_array(m.verts, shape=(nv, 3)).copy()
                     if nv and m.verts else np.zeros((0, 3)))
            return verts, np.zeros((0, 3), dtype=np.int32), np.zeros(0, dtype=np.int32), stats
        verts = np.ctypeslib.as_array(m.verts, shape=(nv, 3)).copy()
        tris = np.ctypeslib.as_array(m.tris, shape=(nt, 3)).copy()
    finally:
        lib().or_mesh_free(ctypes.byref(m))
    return verts, tris, np.full(nt, object_id, dtype=np.int32), stats


def concatenate(meshes):
    """mesh.py:92-105: offsets indices, drops meshes with zero triangles."""
    meshes = [m for m in meshes if len(m[1])]
    if not meshes:
        return np.zeros((0, 3)), np.zeros((0, 3), dtype=np.int32), np.zeros(0, dtype=np.int32)
    verts, tris, oids = [], [], []
    base = 0
    for v, t, o in meshes:
        verts.append(v)
        tris.append(t + base)
        oids.append(o)
        base += len(v)
    return np.concatenate(verts), np.concatenate(tris).astype(np.int32), np.concatenate(oids)


# -------------------------------------------------------------- visibility
def rasterize(verts, tris, cam):
    """visibility.py:34-98 -> (depth (H,W) f64, tri_id (H,W) i32)."""
    verts = np.ascontiguousarray(np.asarray(verts, dtype=np.float64).reshape(-1, 3))
    tris = np.ascontiguousarray(np.asarray(tris, dtype=np.int32).reshape(-1, 3))
    cs = cam_struct([cam])
    depth = np.empty((cam.image_height, cam.image_width))
    tid = np.empty((cam.image_height, cam.image_width), dtype=np.int32)
    lib().or_rasterize(_p(verts), ctypes.c_int64(len(verts)), _p(tris), ctypes.c_int64(len(tris)),
                       _p(cs), _p(depth), _p(tid))
    return depth, tid


def classify(verts, tris, cam, depth, t_v):
    """visibility.py:106-129 -> bool (T,)."""
    verts = np.ascontiguousarray(np.asarray(verts, dtype=np.float64).reshape(-1, 3))
    tris = np.ascontiguousarray(np.asarray(tris, dtype=np.int32).reshape(-1, 3))
    if len(tris) == 0:
        return np.zeros(0, dtype=bool)
    cs = cam_struct([cam])
    depth = np.ascontiguousarray(depth, dtype=np.float64)
    vis = np.zeros(len(tris), dtype=np.uint8)
    lib().or_classify(_p(verts), _p(tris), ctypes.c_int64(len(tris)), _p(cs), _p(depth),
                      ctypes.c_double(t_v), _p(vis))
    return vis.astype(bool)


# ------------------------------------------------------------------ render
def camera_center(cam):
    return -np.asarray(cam.rotation).T @ np.asarray(cam.translation)  # camera.py:61-64


def rank_cameras(virtual, rig):
    """render.py:29-32."""
    keys = sorted((float(np.linalg.norm(camera_center(c) - camera_center(virtual))), c.id)
                  for c in rig)
    return [cid for _, cid in keys]


def triangle_sources(ranking, vis, n_triangles):
    """render.py:35-43."""
    src = np.full(n_triangles, -1, dtype=np.int32)
    unset = np.ones(n_triangles, dtype=bool)
    for cam_id in ranking:
        take = unset & vis[cam_id]
        src[take] = cam_id
        unset &= ~take
    return src


def render_view(verts, tris, rig, frames, vis, virtual, fallback_color=FALLBACK_COLOR):
    """render.py:64-113 -> (color (H,W,3) u8, source (H,W) i32, covered (H,W) bool)."""
    for cam in rig:
        if cam.id not in frames:
            raise ValueError(f"missing frame for camera {cam.id}")
        if cam.id not in vis:
            raise ValueError(f"missing visibility for camera {cam.id}")
    if np.any(np.asarray(virtual.dist) != 0.0):
        raise ValueError("back_project supports zero-distortion cameras only")
    verts = np.ascontiguousarray(np.asarray(verts, dtype=np.float64).reshape(-1, 3))
    tris = np.ascontiguousarray(np.asarray(tris, dtype=np.int32).reshape(-1, 3))
    h, w = virtual.image_height, virtual.image_width
    ranking = rank_cameras(virtual, rig)
    tri_src = triangle_sources(ranking, vis, len(tris))
    cs = cam_struct(rig)
    vs = cam_struct([virtual])
    buf, off = _pack_images([frames[c.id] for c in rig], channels=3)
    color = np.zeros((h, w, 3), dtype=np.uint8)
    source = np.full((h, w), -1, dtype=np.int32)
    covered = np.zeros((h, w), dtype=np.uint8)
    fb = np.ascontiguousarray(np.asarray(fallback_color, dtype=np.uint8).reshape(3))
    ts = np.ascontiguousarray(tri_src) if len(tri_src) else np.zeros(1, dtype=np.int32)
    lib().or_render(_p(verts), ctypes.c_int64(len(verts)), _p(tris), ctypes.c_int64(len(tris)),
                    _p(ts), _p(cs), ctypes.c_int(len(cs)), _p(buf), _p(off), _p(vs), _p(fb),
                    _p(color), _p(source), _p(covered))
    return color, source, covered.astype(bool)


# ---------------------------------------------------------------- pipeline
def run_frame(rig, sils, stage_lo, stage_hi, coarse_spacing, fine_spacing, min_views=1,
              t_small=5, t_large=np.inf, roi_margin=None, t_v=None, iso_mode="exact",
              fixed_isovalue=0.5, keep_depths=False):
    """pipeline.py:115-220 (B-1 .. D-2) -> dict of every stage output."""
    if roi_margin is None:
        roi_margin = coarse_spacing  # pipeline.py:69-70
    if t_v is None:
        t_v = 3.0 * fine_spacing  # pipeline.py:71-72
    out = {"stats": {}}
    st = out["stats"]
    origin, s, dims = grid_from_aabb(stage_lo, stage_hi, coarse_spacing)
    st["sparse_tests"] = dims[0] * dims[1] * dims[2]
    occ = carve(rig, sils, origin, s, dims, min_views)
    st["sparse_occupied"] = int(occ.sum())
    labels, comps = label(occ, dims)
    _, flabels, fcomps = filter_noise(labels, comps, t_small, t_large)
    rois = extract_rois(fcomps, origin, s, dims, roi_margin)
    st["components"] = len(fcomps)
    out.update(coarse=(origin, s, dims, occ), labels=labels, components=comps,
               filtered_labels=flabels, filtered_components=fcomps, rois=rois)
    fine = []
    for lo, hi, _ in rois:
        fo, fs, fd = grid_from_aabb(lo, hi, fine_spacing)
        fine.append((fo, fs, fd, carve(rig, sils, fo, fs, fd, min_views)))
    st["dense_tests"] = sum(g[2][0] * g[2][1] * g[2][2] for g in fine)
    st["dense_occupied"] = sum(int(g[3].sum()) for g in fine)
    out["fine"] = fine
    meshes = []
    fb = inc = 0
    for (lo, hi, cid), (fo, fs, fd, focc) in zip(rois, fine):
        v, t, o, mst = polygonize(focc, fo, fs, fd, rig, sils, iso_mode, fixed_isovalue, cid)
        fb += mst["fallback_edges"]
        inc += mst["inconsistent_starts"]
        meshes.append((v, t, o))
    st["fallback_edges"] = fb
    st["inconsistent_edge_starts"] = inc
    merged = concatenate(meshes)
    st["triangles"] = len(merged[1])
    out["meshes"] = meshes
    out["merged"] = merged
    depths, vis = {}, {}
    for cam in rig:
        depths[cam.id] = rasterize(merged[0], merged[1], cam)[0]
    for cam in rig:
        vis[cam.id] = classify(merged[0], merged[1], cam, depths[cam.id], t_v)
    out["visibility"] = vis
    if keep_depths:
        out["depths"] = depths
    return out


# -------------------------------------------------------------- silhouette
STD_FLOOR = 2.0  # silhouette.py:18


def distance_map(proposal):
    """silhouette.py:59-69."""
    prop = np.ascontiguousarray(np.asarray(proposal, dtype=bool)).view(np.uint8)
    if prop.ndim != 2:
        raise ValueError("proposal mask must be 2D")
    out = np.empty(prop.shape)
    if lib().or_distance_map(_p(prop), ctypes.c_int64(prop.shape[0]),
                             ctypes.c_int64(prop.shape[1]), _p(out)):
        return np.full(prop.shape, np.inf)
    return out


def build_background(frames):
    """silhouette.py:72-87 -> (mean, std) float64 (H, W, C)."""
    if len(frames) < 2:
        raise ValueError("need at least 2 background frames")
    stack = [np.asarray(f) for f in frames]
    stack = [f[:, :, None] if f.ndim == 2 else f for f in stack]
    arr = np.ascontiguousarray(np.stack(stack).astype(np.uint8))
    n = arr[0].size
    mean = np.empty(arr[0].shape)
    std = np.empty(arr[0].shape)
    lib().or_background(_p(arr), ctypes.c_int64(len(arr)), ctypes.c_int64(n), _p(mean), _p(std))
    return mean, std


def extract_silhouette(frame, mean, std, dm, theta_near=3.0, theta_far=8.0, d_max=32.0):
    """silhouette.py:90-109."""
    img = np.asarray(frame)
    if img.ndim == 2:
        img = img[:, :, None]
    img = np.ascontiguousarray(img.astype(np.uint8))
    h, w, c = img.shape
    out = np.zeros((h, w), dtype=np.uint8)
    lib().or_extract(_p(img), _p(np.ascontiguousarray(mean, dtype=np.float64)),
                     _p(np.ascontiguousarray(std, dtype=np.float64)),
                     _p(np.ascontiguousarray(dm, dtype=np.float64)), ctypes.c_int64(h * w),
                     ctypes.c_int64(c), ctypes.c_double(theta_near), ctypes.c_double(theta_far),
                     ctypes.c_double(d_max), _p(out))
    return out.astype(bool)


def rle_runs(occ):
    """voxels.py:100-112 _rle_encode: run lengths of a flat bool array, the
    first run counted as OFF (a leading ON run is preceded by a 0 run)."""
    bits = np.asarray(occ, dtype=bool).reshape(-1)
    n = len(bits)
    if n == 0:
        return np.zeros(0, dtype=np.uint64)
    edges = np.flatnonzero(np.diff(bits.view(np.uint8))) + 1
    bounds = np.concatenate(([0], edges, [n]))
    runs = np.diff(bounds).astype(np.uint64)
    if bits[0]:
        runs = np.concatenate(([np.uint64(0)], runs))
    return runs
