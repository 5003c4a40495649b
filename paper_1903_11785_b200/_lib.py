"""ctypes binding of libfvv.so (the C ABI declared in include/fvv.h).

There is no CPU fallback: if the library is missing or no CUDA device is
present, every hot-path call raises. The library is built in-tree by
``__graft_entry__.build()`` (``make -C paper_1903_11785_b200/csrc``).
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FVV_LIB") or os.path.join(_HERE, "libfvv.so")  # FVV_LIB: experiment builds

FVV_MAX_CAMS = 64
FVV_MAX_GRIDS = 128
FVV_OK, FVV_E_ARG, FVV_E_CUDA, FVV_E_LIMIT = 0, 1, 2, 3

# include/fvv.h fvv_camera (192 bytes)
CAM_DTYPE = np.dtype(
    [
        ("R", "<f8", (9,)), ("t", "<f8", (3,)),
        ("fx", "<f8"), ("fy", "<f8"), ("cx", "<f8"), ("cy", "<f8"), ("skew", "<f8"),
        ("k1", "<f8"), ("k2", "<f8"), ("p1", "<f8"), ("p2", "<f8"), ("k3", "<f8"),
        ("width", "<i4"), ("height", "<i4"), ("id", "<i4"), ("has_distortion", "<i4"),
    ]
)
# include/fvv.h fvv_grid (56 bytes)
GRID_DTYPE = np.dtype([("origin", "<f8", (3,)), ("spacing", "<f8"), ("dims", "<i8", (3,))])
# include/fvv.h fvv_component (64 bytes)
COMP_DTYPE = np.dtype([("id", "<i8"), ("voxel_count", "<i8"), ("bbox_min", "<i8", (3,)),
                       ("bbox_max", "<i8", (3,))])
assert CAM_DTYPE.itemsize == 192 and GRID_DTYPE.itemsize == 56 and COMP_DTYPE.itemsize == 64

# exported symbols; tests check the .so exports every one of them
SYMBOLS = (
    "fvv_last_error", "fvv_version", "fvv_launch_count", "fvv_copy_gather", "fvv_host_mapped",
    "fvv_project", "fvv_pack_silhouettes", "fvv_carve", "fvv_carve_workspace_bytes",
    "fvv_rle_workspace_bytes", "fvv_rle_transitions", "fvv_ccl_workspace_bytes", "fvv_ccl26",
    "fvv_ccl_components", "fvv_ccl_labels", "fvv_filter_labels", "fvv_filter_dense",
    "fvv_mesh_workspace_bytes", "fvv_mesh_prepare", "fvv_mesh_counts",
    "fvv_mesh_emit_scratch_bytes", "fvv_mesh_emit", "fvv_edge_isovalues",
    "fvv_raster_workspace_bytes", "fvv_rasterize", "fvv_rasterize_tracked", "fvv_classify", "fvv_triangle_sources",
    "fvv_render_count", "fvv_render_view", "fvv_render_view_coded", "fvv_back_project",
    "fvv_render_ellipsoids",
    "fvv_frame_create", "fvv_frame_destroy", "fvv_frame_run", "fvv_frame_get_outputs",
    "fvv_frame_last_mode",
    "fvv_frame_set_stage_times",
    "fvv_frame_get_rois", "fvv_frame_readback_layout", "fvv_frame_readback",
    "fvv_synth_render", "fvv_erode_cross", "fvv_distance_map", "fvv_background",
    "fvv_extract_silhouette",
    "fvv_seq_create", "fvv_seq_destroy", "fvv_seq_submit", "fvv_seq_next", "fvv_seq_result_get",
    "fvv_seq_result_free", "fvv_abi_sizes",
)

FRAME_CONFIG_DTYPE = np.dtype([("stage_lo", "<f8", (3,)), ("stage_hi", "<f8", (3,)),
                               ("coarse_spacing", "<f8"), ("fine_spacing", "<f8"),
                               ("roi_margin", "<f8"), ("t_v", "<f8"), ("t_large", "<f8"),
                               ("fixed_isovalue", "<f8"), ("t_small", "<i8"), ("budget", "<i8"),
                               ("min_views", "<i4"), ("exact", "<i4")])
FRAME_STATS_DTYPE = np.dtype([(k, "<i8") for k in (
    "sparse_tests", "sparse_occupied", "components", "dense_tests", "dense_occupied",
    "fallback_edges", "inconsistent_edge_starts", "triangles", "vertices", "n_rois")] +
    [("ms", "<f4", (8,)), ("covered_px", "<i8"), ("sourced_px", "<i8")])


class FrameOutputs(ctypes.Structure):
    _fields_ = [("verts", ctypes.c_void_p), ("tris", ctypes.c_void_p), ("nv", ctypes.c_int64),
                ("nt", ctypes.c_int64), ("vis", ctypes.c_void_p), ("vis_stride", ctypes.c_int64),
                ("depth", ctypes.c_void_p), ("color", ctypes.c_void_p),
                ("source", ctypes.c_void_p), ("covered", ctypes.c_void_p),
                ("n_rois", ctypes.c_int64), ("ntri_dev", ctypes.c_void_p)]


class FrameStats(ctypes.Structure):  # include/fvv.h fvv_frame_stats (128 bytes)
    _fields_ = [(k, ctypes.c_int64) for k in FRAME_STATS_DTYPE.names[:10]] + [
        ("ms", ctypes.c_float * 8), ("covered_px", ctypes.c_int64), ("sourced_px", ctypes.c_int64)]


class SeqConfig(ctypes.Structure):  # include/fvv.h fvv_seq_config
    _fields_ = [("lanes", ctypes.c_int32), ("readback_flags", ctypes.c_int32),
                ("has_virtual", ctypes.c_int32), ("export_payload", ctypes.c_int32),
                ("virt", ctypes.c_uint8 * 192), ("rank_pos", ctypes.c_int32 * FVV_MAX_CAMS),
                ("fallback", ctypes.c_uint8 * 4), ("_pad", ctypes.c_uint8 * 4)]  # C: 8-aligned


class SeqResultInfo(ctypes.Structure):  # include/fvv.h fvv_seq_result_info
    _fields_ = [("id", ctypes.c_int64), ("status", ctypes.c_int32), ("stage", ctypes.c_int32),
                ("err", ctypes.c_char_p), ("stats", FrameStats), ("nv", ctypes.c_int64),
                ("nt", ctypes.c_int64), ("vis_stride", ctypes.c_int64), ("n_rois", ctypes.c_int64),
                ("component_ids", ctypes.c_void_p), ("boxes", ctypes.c_void_p),
                ("grids", ctypes.c_void_p), ("roi_info", ctypes.c_void_p),
                ("layout", ctypes.c_int64 * 16), ("host", ctypes.c_void_p),
                ("payload_dev", ctypes.c_void_p), ("payload_bytes", ctypes.c_int64)]


assert ctypes.sizeof(FrameStats) == FRAME_STATS_DTYPE.itemsize == 128


class FvvError(RuntimeError):
    """A CUDA-side failure reported through the C ABI."""


_lib = None


def load():
    """Load libfvv.so once; raise loudly if it was not built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                "g.build()'` (there is no CPU fallback for the hot path)"
            )
        lib = ctypes.CDLL(LIB_PATH)
        lib.fvv_last_error.restype = ctypes.c_char_p
        lib.fvv_launch_count.restype = ctypes.c_longlong
        lib.fvv_frame_create.restype = ctypes.c_void_p
        lib.fvv_frame_readback_layout.restype = ctypes.c_int64
        lib.fvv_frame_destroy.argtypes = [ctypes.c_void_p]
        lib.fvv_seq_create.restype = ctypes.c_void_p
        lib.fvv_seq_destroy.argtypes = [ctypes.c_void_p]
        lib.fvv_seq_result_free.argtypes = [ctypes.c_void_p]
        lib.fvv_seq_result_get.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
        lib.fvv_seq_next.argtypes = [ctypes.c_void_p, ctypes.c_int,
                                     ctypes.POINTER(ctypes.c_void_p)]
        lib.fvv_seq_submit.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p,
                                       ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]
        lib.fvv_ccl_workspace_bytes.restype = ctypes.c_size_t
        lib.fvv_carve_workspace_bytes.restype = ctypes.c_size_t
        lib.fvv_rle_workspace_bytes.restype = ctypes.c_size_t
        lib.fvv_rle_workspace_bytes.argtypes = [ctypes.c_int64]
        lib.fvv_mesh_workspace_bytes.restype = ctypes.c_size_t
        lib.fvv_mesh_emit_scratch_bytes.restype = ctypes.c_size_t
        lib.fvv_mesh_emit_scratch_bytes.argtypes = [ctypes.c_int64, ctypes.c_int64]
        lib.fvv_raster_workspace_bytes.restype = ctypes.c_size_t
        lib.fvv_raster_workspace_bytes.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_int]
        _lib = lib
    return _lib


def call(name: str, *args) -> None:
    """Invoke an fvv_* entry point and map its status to an exception."""
    rc = getattr(load(), name)(*args)
    if rc != FVV_OK:
        msg = load().fvv_last_error().decode(errors="replace")
        if rc in (FVV_E_ARG, FVV_E_LIMIT):
            raise ValueError(msg)
        raise FvvError(msg)


def host_ptr(a: np.ndarray):
    """Pointer to a host array that keeps the array alive for the call
    (arguments are often temporaries built inline)."""
    p = ctypes.c_void_p(a.ctypes.data)
    p._keep = a
    return p


def dev_ptr(t):
    """Device pointer of a tensor, holding a reference to it."""
    p = ctypes.c_void_p(t.data_ptr())
    p._keep = t
    return p


def i64(v):
    return ctypes.c_int64(int(v))
