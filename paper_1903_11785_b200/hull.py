"""Coarse-to-fine visual hull on the GPU (drop-in for freeview.hull).

B-1 ``carve`` and B-3 ``dense_carve`` run the fvv_carve kernel (one launch
for the stage grid, one launch for all ROI grids); B-2 ``label_components``
runs the fvv_ccl26 union-find kernels and ``filter_noise`` the fvv_filter
kernel. ``extract_rois`` is host bookkeeping over the (few) components,
computed with the reference's numpy expressions (hull.py:272-284).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._device import DeviceSilhouettes, grid_table, require_cuda, stream_handle, words_for
from .voxels import DEFAULT_VOXEL_BUDGET, GridSpec, VoxelGrid

CARVE_CHUNK = 1 << 20  # hull.py:20 (kept for API parity; the GPU carves all voxels at once)


@dataclass
class Component:
    """hull.py:23-28."""

    id: int
    voxel_count: int
    bbox_min: tuple  # inclusive (i, j, k)
    bbox_max: tuple


@dataclass
class Labeling:
    """hull.py:31-34; ``labels`` is materialised from the GPU on first read."""

    labels: np.ndarray
    components: list


@dataclass
class NoiseFilterParams:
    """hull.py:37-47: keep components with t_small <= count <= t_large."""

    t_small: int = 0
    t_large: float = np.inf

    def __post_init__(self) -> None:
        if not (0 <= self.t_small <= self.t_large):
            raise ValueError("require 0 <= t_small <= t_large")

    def keeps(self, count: int) -> bool:
        return self.t_small <= count <= self.t_large


@dataclass
class Roi:
    """hull.py:50-60: world-space AABB of one component."""

    lo: np.ndarray
    hi: np.ndarray
    component_id: int

    def __post_init__(self) -> None:
        self.lo = np.asarray(self.lo, dtype=np.float64).reshape(3)
        self.hi = np.asarray(self.hi, dtype=np.float64).reshape(3)
        if (self.lo >= self.hi).any():
            raise ValueError("ROI must have positive extent")


def _as_device_sils(rig, sils) -> DeviceSilhouettes:
    if isinstance(sils, DeviceSilhouettes):
        if sils.ncam != len(rig):
            raise ValueError(f"{sils.ncam} silhouettes for {len(rig)} cameras")
        return sils
    return DeviceSilhouettes(rig, sils)


def carve_grids(dsils: DeviceSilhouettes, specs, min_views: int = 1):
    """Carve every grid of ``specs`` in one fvv_carve launch per
    FVV_MAX_GRIDS batch. Returns VoxelGrids backed by views into one device
    bit buffer; ON counts stay on the device until asked for."""
    specs = list(specs)
    dev = dsils.device
    words = [words_for(s.num_voxels) for s in specs]
    word_off = np.zeros(len(specs), dtype=np.int64)
    if specs:
        word_off[1:] = np.cumsum(words)[:-1]
    bits = torch.empty(max(int(sum(words)), 1), dtype=torch.int32, device=dev)
    counts = torch.zeros(max(len(specs), 1), dtype=torch.int64, device=dev)
    for b0 in range(0, len(specs), _lib.FVV_MAX_GRIDS):
        chunk = specs[b0:b0 + _lib.FVV_MAX_GRIDS]
        tab = grid_table(chunk)
        off = np.ascontiguousarray(word_off[b0:b0 + len(chunk)])
        _lib.call("fvv_carve", _lib.host_ptr(dsils.cams), ctypes.c_int(dsils.ncam),
                  _lib.dev_ptr(dsils.bits), _lib.host_ptr(dsils.word_off), _lib.host_ptr(tab),
                  ctypes.c_int(len(chunk)), _lib.host_ptr(off), ctypes.c_int(int(min_views)),
                  _lib.dev_ptr(bits), _lib.dev_ptr(counts[b0:]), stream_handle())
    return [VoxelGrid(s, bits=bits[int(o):int(o) + w], count=counts[g])
            for g, (s, o, w) in enumerate(zip(specs, word_off, words))]


def carve(rig, sils, spec: GridSpec, min_views: int = 1, workers: int = 1) -> VoxelGrid:
    """Silhouette-consistency carve (hull.py:95-119) on the GPU.

    A voxel is ON iff its centre is in-frustum for at least ``min_views``
    cameras and every camera that sees it observes foreground at the
    rounded pixel. ``workers`` is accepted for API parity and ignored."""
    dsils = _as_device_sils(rig, sils)
    return carve_grids(dsils, [spec], min_views)[0]


def dense_carve(rig, sils, rois, fine_spacing: float, min_views: int = 1, workers: int = 1,
                budget: int = None) -> list:
    """Per-ROI fine carve (hull.py:287-302), all ROIs in one launch."""
    kw = {} if budget is None else {"budget": budget}
    specs = [GridSpec.from_aabb(r.lo, r.hi, fine_spacing, **kw) for r in rois]
    if not specs:
        return []
    return carve_grids(_as_device_sils(rig, sils), specs, min_views)


def extract_rois(lab: Labeling, spec: GridSpec, margin: float) -> list:
    """Margin-expanded, stage-clamped world AABB per component (hull.py:272-284)."""
    stage_lo, stage_hi = spec.origin, spec.extent
    out = []
    for c in lab.components:
        lo = spec.origin + spec.spacing * np.asarray(c.bbox_min, dtype=np.float64) - margin
        hi = spec.origin + spec.spacing * (np.asarray(c.bbox_max, dtype=np.float64) + 1.0) + margin
        out.append(Roi(lo=np.maximum(lo, stage_lo), hi=np.minimum(hi, stage_hi),
                       component_id=c.id))
    return out
