"""Adaptive background subtraction on the GPU (drop-in for freeview.silhouette).

The upstream producer of the hot path's silhouettes:
``distance_map`` (exact EDT of the proposal mask, fvv_distance_map),
``build_background`` (per-pixel mean / population std with a floor,
fvv_background) and ``extract_silhouette`` (max-over-channels normalised
deviation against the distance-ramped threshold, fvv_extract_silhouette).
Results equal the reference's scipy/numpy ones bit for bit.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._device import require_cuda, stream_handle

STD_FLOOR = 2.0  # silhouette.py:18


@dataclass
class BackgroundModel:
    """silhouette.py:21-29 (mean/std float64 (H, W, C)); a device copy is kept
    for the extraction kernel."""

    mean: np.ndarray
    std: np.ndarray

    @property
    def shape(self):
        return self.mean.shape

    def device(self):
        d = getattr(self, "_dev", None)
        if d is None:
            dev = require_cuda()
            d = (torch.from_numpy(np.ascontiguousarray(self.mean, dtype=np.float64)).to(dev),
                 torch.from_numpy(np.ascontiguousarray(self.std, dtype=np.float64)).to(dev))
            self._dev = d
        return d


@dataclass
class AdaptiveParams:
    """silhouette.py:32-47."""

    theta_near: float = 3.0
    theta_far: float = 8.0
    d_max: float = 32.0

    def __post_init__(self) -> None:
        if not (0 < self.theta_near <= self.theta_far):
            raise ValueError("require 0 < theta_near <= theta_far")
        if self.d_max <= 0:
            raise ValueError("d_max must be positive")

    def threshold(self, d):
        """Host helper: the ramp the extraction kernel applies per pixel."""
        t = np.minimum(np.asarray(d, dtype=np.float64) / self.d_max, 1.0)
        return self.theta_near + (self.theta_far - self.theta_near) * t


def _channels(img) -> np.ndarray:
    a = np.asarray(img)
    if a.ndim == 2:
        a = a[:, :, None]
    if a.ndim != 3:
        raise ValueError(f"expected (H, W) or (H, W, C) image, got shape {a.shape}")
    return a


def _u8(t, dev):
    if isinstance(t, torch.Tensor):
        return t.to(dev, non_blocking=True).contiguous()
    return torch.from_numpy(np.ascontiguousarray(np.asarray(t).astype(np.uint8))).to(dev)


def distance_map_device(prop_dev, h, w):
    """(squared distances int32, dm float64) CUDA tensors for one proposal."""
    dev = prop_dev.device
    sq = torch.empty((h, w), dtype=torch.int32, device=dev)
    dm = torch.empty((h, w), dtype=torch.float64, device=dev)
    ws = torch.empty((h, w), dtype=torch.int32, device=dev)
    _lib.call("fvv_distance_map", _lib.dev_ptr(prop_dev), _lib.i64(h), _lib.i64(w),
              _lib.dev_ptr(sq), _lib.dev_ptr(dm), _lib.dev_ptr(ws), stream_handle())
    return sq, dm


def distance_map(proposal) -> np.ndarray:
    """Exact Euclidean distance (px) to the nearest proposal pixel: 0 on the
    proposal, +inf everywhere when it is empty (silhouette.py:59-69)."""
    prop = np.asarray(proposal, dtype=bool)
    if prop.ndim != 2:
        raise ValueError("proposal mask must be 2D")
    dev = require_cuda()
    d_prop = torch.from_numpy(np.ascontiguousarray(prop).view(np.uint8)).to(dev)
    return distance_map_device(d_prop, *prop.shape)[1].cpu().numpy()


def build_background(frames) -> BackgroundModel:
    """Per-pixel, per-channel mean / population std over object-free frames,
    std floored at STD_FLOOR (silhouette.py:72-87)."""
    if len(frames) < 2:
        raise ValueError("need at least 2 background frames")
    stack = [_channels(f) for f in frames]
    shape = stack[0].shape
    for idx, f in enumerate(stack):
        if f.shape != shape:
            raise ValueError(f"frame {idx} shape {f.shape} != {shape}")
    dev = require_cuda()
    d_frames = torch.from_numpy(np.ascontiguousarray(np.stack(stack).astype(np.uint8))).to(dev)
    n = int(np.prod(shape))
    mean = torch.empty(shape, dtype=torch.float64, device=dev)
    std = torch.empty(shape, dtype=torch.float64, device=dev)
    _lib.call("fvv_background", _lib.dev_ptr(d_frames), _lib.i64(len(stack)), _lib.i64(n),
              _lib.dev_ptr(mean), _lib.dev_ptr(std), stream_handle())
    bg = BackgroundModel(mean=mean.cpu().numpy(), std=std.cpu().numpy())
    bg._dev = (mean, std)
    return bg


def extract_device(frame_dev, bg: BackgroundModel, dm_dev, params: AdaptiveParams, sq_dev=None):
    """uint8 (H, W) silhouette mask on the GPU."""
    mean, std = bg.device()
    h, w, c = bg.shape
    out = torch.empty((h, w), dtype=torch.uint8, device=mean.device)
    _lib.call("fvv_extract_silhouette", _lib.dev_ptr(frame_dev), _lib.dev_ptr(mean),
              _lib.dev_ptr(std), _lib.i64(h * w), ctypes.c_int(c),
              _lib.dev_ptr(sq_dev) if sq_dev is not None else ctypes.c_void_p(0),
              _lib.dev_ptr(dm_dev) if dm_dev is not None else ctypes.c_void_p(0),
              ctypes.c_double(params.theta_near), ctypes.c_double(params.theta_far),
              ctypes.c_double(params.d_max), _lib.dev_ptr(out), stream_handle())
    return out


def extract_silhouette(frame, bg: BackgroundModel, dm, params: AdaptiveParams) -> np.ndarray:
    """Foreground iff the max-over-channels normalised deviation exceeds the
    distance-adapted threshold (silhouette.py:90-109)."""
    img = _channels(frame)
    if img.shape != bg.shape:
        raise ValueError(f"frame shape {img.shape} != background shape {bg.shape}")
    dm = np.asarray(dm, dtype=np.float64)
    if dm.shape != img.shape[:2]:
        raise ValueError(f"distance map shape {dm.shape} != frame shape {img.shape[:2]}")
    dev = require_cuda()
    d_img = _u8(img, dev)
    d_dm = torch.from_numpy(np.ascontiguousarray(dm)).to(dev)
    return extract_device(d_img, bg, d_dm, params).cpu().numpy().astype(bool)


def silhouettes_device(rig, frames, proposals, background, params: AdaptiveParams):
    """Every camera's silhouette (pipeline.py:104-112 compute_silhouettes) as
    one uint8 (N*H*W,) CUDA tensor in rig order, computed on the GPU."""
    dev = require_cuda()
    cams = list(rig)
    parts = []
    for cam in cams:
        prop = proposals[cam.id]
        if isinstance(prop, torch.Tensor):
            d_prop = prop.to(dev).view(torch.uint8) if prop.dtype == torch.bool else \
                prop.to(dev)
        else:
            p = np.asarray(prop, dtype=bool)
            if p.ndim != 2:
                raise ValueError("proposal mask must be 2D")
            d_prop = torch.from_numpy(np.ascontiguousarray(p).view(np.uint8)).to(dev)
        h, w = d_prop.shape
        sq, _ = distance_map_device(d_prop.contiguous(), h, w)
        bg = background[cam.id]
        img = frames[cam.id]
        shape = tuple(img.shape) if isinstance(img, torch.Tensor) else _channels(img).shape
        if len(shape) == 2:
            shape = (*shape, 1)
        if tuple(shape) != tuple(bg.shape):
            raise ValueError(f"frame shape {tuple(shape)} != background shape {bg.shape}")
        if (h, w) != tuple(bg.shape[:2]):
            raise ValueError(f"distance map shape {(h, w)} != frame shape {bg.shape[:2]}")
        parts.append(extract_device(_u8(img, dev), bg, None, params, sq_dev=sq).reshape(-1))
    return torch.cat(parts)
