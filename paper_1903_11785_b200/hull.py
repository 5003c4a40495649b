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


class Labeling:
    """hull.py:31-34: flat int32 ``labels`` (0 = background) and the
    ``components`` list (ascending id).

    A labelling produced on the GPU keeps its labels in device memory (the
    CCL workspace, or a dense device array after filtering) and copies them
    to the host only when ``labels`` is read."""

    def __init__(self, labels=None, components=None, *, spec=None, ws=None, dense=None):
        self.components = list(components or [])
        self._labels = None if labels is None else np.asarray(labels, dtype=np.int32)
        self._spec = spec
        self._ws = ws
        self._dense = dense

    @property
    def labels(self) -> np.ndarray:
        if self._labels is None:
            self._labels = self.device_labels().cpu().numpy()
        return self._labels

    @labels.setter
    def labels(self, value) -> None:
        self._labels = np.asarray(value, dtype=np.int32)
        self._ws = self._dense = None

    def device_labels(self) -> torch.Tensor:
        """Dense int32 labels on the GPU."""
        if self._dense is None:
            if self._ws is not None:
                n = self._spec.num_voxels
                dense = torch.empty(n, dtype=torch.int32, device=self._ws.device)
                _lib.call("fvv_ccl_labels", _lib.host_ptr(grid_table([self._spec])),
                          _lib.dev_ptr(self._ws), _lib.dev_ptr(dense), stream_handle())
                self._dense = dense
            else:
                self._dense = torch.from_numpy(self._labels).to(require_cuda())
        return self._dense

    def __repr__(self) -> str:
        return f"Labeling(components={self.components!r})"


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
    ws_bytes = int(_lib.load().fvv_carve_workspace_bytes(_lib.host_ptr(dsils.cams),
                                                         ctypes.c_int(dsils.ncam)))
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)  # stream-ordered reuse
    for b0 in range(0, len(specs), _lib.FVV_MAX_GRIDS):
        chunk = specs[b0:b0 + _lib.FVV_MAX_GRIDS]
        tab = grid_table(chunk)
        off = np.ascontiguousarray(word_off[b0:b0 + len(chunk)])
        _lib.call("fvv_carve", _lib.host_ptr(dsils.cams), ctypes.c_int(dsils.ncam),
                  _lib.dev_ptr(dsils.bits), _lib.host_ptr(dsils.word_off), _lib.host_ptr(tab),
                  ctypes.c_int(len(chunk)), _lib.host_ptr(off), ctypes.c_int(int(min_views)),
                  _lib.dev_ptr(bits), _lib.dev_ptr(counts[b0:]), _lib.dev_ptr(ws),
                  ctypes.c_size_t(ws_bytes), stream_handle())
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


def _comps_from_records(rec) -> list:
    return [Component(id=int(r["id"]), voxel_count=int(r["voxel_count"]),
                      bbox_min=tuple(int(v) for v in r["bbox_min"]),
                      bbox_max=tuple(int(v) for v in r["bbox_max"])) for r in rec]


_COMP_PREFETCH = 4096  # component records copied back with the counts (one sync)


def label_grid_async(grid: VoxelGrid):
    """Launch fvv_ccl26 on ``grid``; returns (workspace, comps_dev, counts_dev)
    without synchronising."""
    dev = require_cuda()
    tab = grid_table([grid.spec])
    nbytes = int(_lib.load().fvv_ccl_workspace_bytes(_lib.host_ptr(tab)))
    ws = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    comps = torch.empty((_COMP_PREFETCH, _lib.COMP_DTYPE.itemsize), dtype=torch.uint8, device=dev)
    counts = torch.zeros(2, dtype=torch.int64, device=dev)
    _lib.call("fvv_ccl26", _lib.dev_ptr(grid.device_bits(dev)), _lib.host_ptr(tab),
              _lib.dev_ptr(ws), ctypes.c_size_t(nbytes), _lib.dev_ptr(comps),
              _lib.i64(_COMP_PREFETCH), _lib.dev_ptr(counts), stream_handle())
    return ws, comps, counts


def finish_labels(grid: VoxelGrid, ws, comps, counts) -> Labeling:
    """Read the component table back (one sync) and wrap the labelling."""
    n_on, ncomp = (int(v) for v in counts.cpu().tolist())
    if ncomp > _COMP_PREFETCH:
        comps = torch.empty((ncomp, _lib.COMP_DTYPE.itemsize), dtype=torch.uint8,
                            device=ws.device)
        _lib.call("fvv_ccl_components", _lib.host_ptr(grid_table([grid.spec])),
                  _lib.dev_ptr(ws), _lib.dev_ptr(comps), _lib.i64(ncomp), stream_handle())
    rec = comps[:ncomp].cpu().numpy().view(_lib.COMP_DTYPE).reshape(-1)
    return Labeling(components=_comps_from_records(rec), spec=grid.spec, ws=ws)


def label_components(grid: VoxelGrid, block_dims=(16, 16, 16)) -> Labeling:
    """26-connected components labelling on the GPU (hull.py:218-254).

    Ids 1..n ascend with each component's minimum linear voxel index, as in
    the reference. ``block_dims`` is validated for API parity; the GPU
    union-find's result does not depend on any decomposition (nor does the
    reference's)."""
    bx, by, bz = (int(b) for b in block_dims)
    if min(bx, by, bz) < 1:
        raise ValueError("block dims must be >= 1")
    return finish_labels(grid, *label_grid_async(grid))


def filter_noise(grid: VoxelGrid, lab: Labeling, params: NoiseFilterParams):
    """Drop components whose voxel count is outside [t_small, t_large]
    (hull.py:257-269); survivors keep their ids and voxels. Runs the
    fvv_filter kernel over the device labelling."""
    dev = require_cuda()
    kept = [c for c in lab.components if params.keeps(c.voxel_count)]
    keep = np.zeros(len(lab.components) + 1, dtype=np.uint8)
    keep[[c.id for c in kept]] = 1
    keep_d = torch.from_numpy(keep).to(dev)
    n = grid.spec.num_voxels
    labels = torch.empty(n, dtype=torch.int32, device=dev)
    bits = torch.empty(max(words_for(n), 1), dtype=torch.int32, device=dev)
    count = torch.zeros(1, dtype=torch.int64, device=dev)
    if lab._ws is not None and lab._spec is not None and lab._spec.num_voxels == n:
        _lib.call("fvv_filter_labels", _lib.host_ptr(grid_table([grid.spec])),
                  _lib.dev_ptr(lab._ws), _lib.dev_ptr(keep_d), _lib.dev_ptr(labels),
                  _lib.dev_ptr(bits), _lib.dev_ptr(count), stream_handle())
    else:
        src = lab.device_labels()
        _lib.call("fvv_filter_dense", _lib.dev_ptr(src), _lib.i64(n), _lib.dev_ptr(keep_d),
                  _lib.i64(len(keep)), _lib.dev_ptr(labels), _lib.dev_ptr(bits),
                  _lib.dev_ptr(count), stream_handle())
    return (VoxelGrid(grid.spec, bits=bits, count=count[0]),
            Labeling(components=kept, spec=grid.spec, dense=labels))


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
