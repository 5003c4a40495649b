"""Device plumbing: CUDA device/stream handles, camera tables and resident
silhouette bit-planes. PyTorch only allocates device memory and supplies
streams; every computation goes through libfvv.so."""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib


def require_cuda() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("the freeview B200 path needs a CUDA device (no CPU fallback)")
    _lib.load()
    return torch.device("cuda", torch.cuda.current_device())


def stream_handle():
    """The current CUDA stream of the current device (raw handle: a tenth of
    torch.cuda.current_stream()'s cost, which is paid on every frame)."""
    raw = getattr(torch._C, "_cuda_getCurrentRawStream", None)
    if raw is not None:
        return ctypes.c_void_p(raw(torch.cuda.current_device()))
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


_CAM_CACHE = {}


def _cam_key(c):
    return (int(c.id), int(c.image_width), int(c.image_height), float(c.fx), float(c.fy),
            float(c.cx), float(c.cy), float(c.skew),
            np.asarray(c.dist, dtype=np.float64).tobytes(),
            np.asarray(c.rotation, dtype=np.float64).tobytes(),
            np.asarray(c.translation, dtype=np.float64).tobytes())


def cam_table(cams) -> np.ndarray:
    """CameraModel-like objects -> fvv_camera records (include/fvv.h),
    memoised on the cameras' parameter values (rigs are reused every frame)."""
    cams = list(cams)
    key = tuple(_cam_key(c) for c in cams)
    hit = _CAM_CACHE.get(key)
    if hit is not None:
        return hit
    out = _build_cam_table(cams)
    if len(_CAM_CACHE) > 256:
        _CAM_CACHE.clear()
    out.setflags(write=False)
    _CAM_CACHE[key] = out
    return out


def _build_cam_table(cams) -> np.ndarray:
    out = np.zeros(len(cams), dtype=_lib.CAM_DTYPE)
    for i, c in enumerate(cams):
        dist = np.asarray(c.dist, dtype=np.float64).reshape(5)
        out[i]["R"] = np.asarray(c.rotation, dtype=np.float64).reshape(9)
        out[i]["t"] = np.asarray(c.translation, dtype=np.float64).reshape(3)
        out[i]["fx"], out[i]["fy"] = float(c.fx), float(c.fy)
        out[i]["cx"], out[i]["cy"], out[i]["skew"] = float(c.cx), float(c.cy), float(c.skew)
        out[i]["k1"], out[i]["k2"], out[i]["p1"], out[i]["p2"], out[i]["k3"] = dist
        out[i]["width"], out[i]["height"] = int(c.image_width), int(c.image_height)
        out[i]["id"] = int(c.id)
        out[i]["has_distortion"] = int(bool(np.any(dist != 0.0)))
    return out


def grid_table(specs) -> np.ndarray:
    specs = list(specs)
    out = np.zeros(len(specs), dtype=_lib.GRID_DTYPE)
    for i, s in enumerate(specs):
        out[i]["origin"] = np.asarray(s.origin, dtype=np.float64)
        out[i]["spacing"] = float(s.spacing)
        out[i]["dims"] = np.asarray(s.dims, dtype=np.int64)
    return out


def words_for(nvox: int) -> int:
    return (int(nvox) + 31) // 32


def bits_to_bool(bits: torch.Tensor, nvox: int) -> np.ndarray:
    """Occupancy words (device int32 view) -> flat numpy bool[nvox]."""
    raw = bits.cpu().numpy().view(np.uint8)
    return np.unpackbits(raw, bitorder="little")[:nvox].astype(bool)


def bool_to_bits(occ: np.ndarray, device) -> torch.Tensor:
    occ = np.asarray(occ, dtype=bool).reshape(-1)
    nw = words_for(len(occ))
    packed = np.zeros(nw * 4, dtype=np.uint8)
    p = np.packbits(occ, bitorder="little")
    packed[: len(p)] = p
    return torch.from_numpy(packed.view(np.int32)).to(device)


def mask_bytes(t):
    """Silhouette tensor -> one byte per pixel, nonzero = foreground (the
    packing kernel's reading). bool/uint8/int8 are reinterpreted in place;
    any other dtype is compared with zero, as np.asarray(sil, dtype=bool)
    does in hull.py:68."""
    if t.dtype == torch.bool or t.dtype == torch.int8:
        return t.view(torch.uint8)
    if t.dtype == torch.uint8:
        return t
    return (t != 0).to(torch.uint8)


class DeviceSilhouettes:
    """Bit-packed silhouettes of a rig, resident on the GPU.

    Validates like hull.py:63-75 (_check_sils), uploads the masks once and
    packs them with fvv_pack_silhouettes; every kernel of the frame reads
    these bit-planes (4.15 MB for 16 x 1080p, L2-resident)."""

    def __init__(self, rig, sils, device=None):
        device = device or require_cuda()
        cams = list(rig)
        if len(sils) != len(cams):
            raise ValueError(f"{len(sils)} silhouettes for {len(cams)} cameras")
        if len(cams) > _lib.FVV_MAX_CAMS:
            raise ValueError(f"{len(cams)} cameras exceed the kernel limit {_lib.FVV_MAX_CAMS}")
        self.cams = cam_table(cams)
        self.ncam = len(cams)
        sizes = [c.image_height * c.image_width for c in cams]
        self.mask_off = np.zeros(self.ncam, dtype=np.int64)
        self.mask_off[1:] = np.cumsum(sizes)[:-1]
        words = [c.image_height * ((c.image_width + 31) // 32) for c in cams]
        self.word_off = np.zeros(self.ncam, dtype=np.int64)
        self.word_off[1:] = np.cumsum(words)[:-1]
        total_words = int(sum(words))

        if isinstance(sils, torch.Tensor) and sils.dim() == 3:
            shape = tuple(sils.shape[1:])
            for c in cams:
                if shape != (c.image_height, c.image_width):
                    raise ValueError(
                        f"camera {c.id}: silhouette shape {shape} != "
                        f"({c.image_height}, {c.image_width})")
            masks = mask_bytes(sils.reshape(-1)).to(device, non_blocking=True)
        else:
            host = []
            for c, s in zip(cams, sils):
                if isinstance(s, torch.Tensor):
                    s = s.cpu().numpy()
                s = np.asarray(s)
                if s.shape != (c.image_height, c.image_width):
                    raise ValueError(
                        f"camera {c.id}: silhouette shape {s.shape} != "
                        f"({c.image_height}, {c.image_width})")
                host.append(np.ascontiguousarray(s if s.dtype == np.bool_ else s.astype(bool)))
            masks = torch.empty(int(sum(sizes)), dtype=torch.uint8, device=device)
            for h, off, sz in zip(host, self.mask_off, sizes):
                masks[int(off):int(off) + sz].copy_(
                    torch.from_numpy(h.reshape(-1).view(np.uint8)), non_blocking=False)
        self.bits = torch.empty(max(total_words, 1), dtype=torch.int32, device=device)
        _lib.call("fvv_pack_silhouettes", _lib.host_ptr(self.cams), ctypes.c_int(self.ncam),
                  _lib.dev_ptr(masks), _lib.host_ptr(self.mask_off), _lib.dev_ptr(self.bits),
                  _lib.host_ptr(self.word_off), stream_handle())
        self._masks = masks  # keep alive until the pack kernel has run
        self.device = device
