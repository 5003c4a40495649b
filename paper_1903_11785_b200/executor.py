"""Python face of the native frame executor (fvv_frame_*, csrc/frame.cu).

One executor per (rig, PipelineConfig): the C++ side runs B-1 .. D-2 and the
optional virtual-view colour pass on the current CUDA stream with device
buffers that persist across frames; Python only hands over the inputs and
wraps the outputs. ``FrameExecutor.run`` returns a ``FrameOutput`` whose
device views stay valid until the executor's next run; ``to_host`` copies
everything a SceneBundle needs back in one batch of pinned transfers.
"""

from __future__ import annotations

import ctypes
from collections import OrderedDict

import numpy as np
import torch

from . import _lib
from ._device import cam_table, mask_bytes, require_cuda, stream_handle

STAGE_NAMES = {1: "B-1 sparse carve", 2: "B-2 noise filter/ROI", 3: "B-3 dense carve",
               4: "C polygonize", 5: "D-1 depth images", 6: "D-2 visibility",
               7: "E render view", 8: "D-2 visibility"}
_INFO_VBASE, _INFO_V, _INFO_SBASE, _INFO_S, _INFO_TBASE, _INFO_T, _INFO_FB, _INFO_INC = range(8)


class _CudaView:
    """Minimal __cuda_array_interface__ over executor-owned device memory."""

    def __init__(self, ptr, shape, typestr):
        self.__cuda_array_interface__ = {"shape": tuple(int(s) for s in shape),
                                         "typestr": typestr, "data": (int(ptr or 0), False),
                                         "version": 3, "strides": None}


def _dev(ptr, shape, typestr):
    if not ptr or 0 in shape:
        return torch.empty(shape, dtype={"<f8": torch.float64, "<i4": torch.int32,
                                         "<u4": torch.int32, "|u1": torch.uint8,
                                         "<i8": torch.int64}[typestr], device="cuda")
    t = torch.as_tensor(_CudaView(ptr, shape, typestr), device="cuda")
    return t.view(torch.int32) if typestr == "<u4" else t


_READBACK_NAMES = ("verts", "tris", "vis", "color", "source", "covered", "depth")


class FrameOutput:
    """Results of one executor run: host scalars, and device views (built on
    first access) that stay valid until the executor's next run."""

    def __init__(self, stats, outs, rois, ncam, virtual, handle=None, owner=None):
        self._owner = owner  # the FrameExecutor owning the device buffers: keep it alive
        self.stats_raw = stats
        self._outs = outs
        self._h = handle
        self.ncam = ncam
        self.virtual = virtual
        self.nv, self.nt = int(outs.nv), int(stats["triangles"])
        self.vis_stride = int(outs.vis_stride)
        self.component_ids, self.boxes, self.grids, self.info = rois

    @property
    def verts(self):
        return _dev(self._outs.verts, (self.nv, 3), "<f8")

    @property
    def tris(self):
        return _dev(self._outs.tris, (self.nt, 3), "<i4")

    @property
    def vis_bits(self):
        return _dev(self._outs.vis, (self.ncam, self.vis_stride), "<u4")

    @property
    def ntri_dev(self):
        return _dev(self._outs.ntri_dev, (1,), "<i8") if self._outs.ntri_dev else None

    @property
    def image(self):
        if self.virtual is None:
            return None
        h, w = self.virtual.image_height, self.virtual.image_width
        o = self._outs
        return (_dev(o.color, (h, w, 3), "|u1"), _dev(o.source, (h, w), "<i4"),
                _dev(o.covered, (h, w), "|u1"))

    def stats(self) -> dict:
        s = self.stats_raw
        return {k: int(s[k]) for k in ("sparse_tests", "sparse_occupied", "components",
                                       "dense_tests", "dense_occupied", "fallback_edges",
                                       "inconsistent_edge_starts", "triangles")}

    def to_host_async(self, cams, keep_depths=False, stream=None, compact=False,
                      image_only=False):
        """Queue the D2H copy of vertices, triangles, visibility bits, the
        rendered image (and depth planes) into ONE pinned block on ``stream``
        (default: the current stream, after this frame's work) with one
        fvv_frame_readback call. Must be called before the executor's next
        run. Returns (HostBlock, completion event)."""
        cur = torch.cuda.current_stream()
        stream = stream or cur
        if stream is not cur:
            stream.wait_stream(cur)
        lib = _lib.load()
        lay = np.zeros(16, dtype=np.int64)
        compact = bool(compact and self.virtual is not None)
        flags = ctypes.c_int(int(bool(keep_depths)) | (2 if compact else 0) |
                             (4 if image_only else 0))
        total = int(lib.fvv_frame_readback_layout(self._h, flags, _lib.host_ptr(lay)))
        buf = torch.empty(max(total, 1), dtype=torch.uint8, pin_memory=True)
        _lib.call("fvv_frame_readback", self._h, ctypes.c_void_p(buf.data_ptr()), flags,
                  ctypes.c_void_p(stream.cuda_stream))
        ev = torch.cuda.Event()
        ev.record(stream)
        return HostBlock(self, buf, lay, keep_depths, compact, image_only), ev

    def export(self, device):
        """(meta float64 array, device uint8 payload) of this frame's mesh
        and visibility bits in the frame-export format (sharding.py), copied
        on the current stream so the executor may run its next frame at once."""
        from .sharding import export_meta, payload_layout

        meta = export_meta(self.stats(), self.stats_raw["ms"][:6], self.component_ids,
                           self.info, self.nv, self.nt, self.ncam, self.vis_stride)
        offs, total = payload_layout(self.nv, self.nt, self.ncam, self.vis_stride)
        payload = torch.empty(max(total, 1), dtype=torch.uint8, device=device)
        for (off, n), src in zip(offs, (self.verts, self.tris, self.vis_bits)):
            if n:
                payload[off:off + n].copy_(src.reshape(-1).view(torch.uint8))
        return meta, payload

    def to_host(self, cams, keep_depths=False):
        """Pinned D2H of every host-facing output, one synchronisation."""
        block, ev = self.to_host_async(cams, keep_depths)
        ev.synchronize()
        return block.arrays()


class HostBlock:
    """One frame's outputs in a pinned host block (executor readback layout)."""

    def __init__(self, out, buf, lay, keep_depths, compact=False, image_only=False):
        self.buf, self.lay = buf, lay
        self.nbytes = int(sum(int(lay[8 + i]) for i in range(7)))  # bytes copied
        self.shapes = {} if image_only else {
            "verts": ((out.nv, 3), np.float64), "tris": ((out.nt, 3), np.int32),
            "vis": ((out.ncam, out.vis_stride), np.uint32)}
        if out.virtual is not None:
            h, w = out.virtual.image_height, out.virtual.image_width
            if compact:  # slot 4: int8 code plane (fvv_frame_readback flag bit 1)
                self.shapes.update(color=((h, w, 3), np.uint8), code=((h, w), np.int8))
            else:
                self.shapes.update(color=((h, w, 3), np.uint8), source=((h, w), np.int32),
                                   covered=((h, w), np.uint8))
        if keep_depths and out.nt:
            self.shapes["depth"] = ((int(lay[14]) // 8,), np.float64)

    def arrays(self) -> dict:
        raw = self.buf.numpy()
        out = {}
        for i, name in enumerate(_READBACK_NAMES):
            if name == "source" and "code" in self.shapes:
                name = "code"
            if name not in self.shapes:
                continue
            shape, dt = self.shapes[name]
            off, n = int(self.lay[i]), int(self.lay[8 + i])
            out[name] = raw[off:off + n].view(dt).reshape(shape)
        return out


def frame_config(cfg, budget) -> np.ndarray:
    """PipelineConfig -> include/fvv.h fvv_frame_config record."""
    conf = np.zeros(1, dtype=_lib.FRAME_CONFIG_DTYPE)
    conf["stage_lo"] = np.asarray(cfg.stage_lo, dtype=np.float64)
    conf["stage_hi"] = np.asarray(cfg.stage_hi, dtype=np.float64)
    conf["coarse_spacing"] = cfg.coarse_spacing
    conf["fine_spacing"] = cfg.fine_spacing
    conf["roi_margin"] = cfg.roi_margin
    conf["t_v"] = cfg.t_v
    conf["t_large"] = float(cfg.t_large)
    conf["fixed_isovalue"] = cfg.fixed_isovalue
    conf["t_small"] = int(cfg.t_small)
    conf["budget"] = int(budget)
    conf["min_views"] = int(cfg.min_views)
    conf["exact"] = int(cfg.iso_mode == "exact")
    return conf


_FALLBACK_PTR = []


def _fallback_ptr():
    """Pointer to render.py's fallback colour (built once)."""
    if not _FALLBACK_PTR:
        from .render import FALLBACK_COLOR

        _FALLBACK_PTR.append(_lib.host_ptr(np.ascontiguousarray(
            np.asarray(FALLBACK_COLOR, dtype=np.uint8).reshape(3))))
    return _FALLBACK_PTR[0]


class FrameExecutor:
    """fvv_frame handle for one rig + PipelineConfig."""

    def __init__(self, cfg, rig, budget=None):
        from .voxels import DEFAULT_VOXEL_BUDGET

        require_cuda()
        self.cams = list(rig)
        self.ncam = len(self.cams)
        self._tab = cam_table(self.cams)
        conf = frame_config(cfg, DEFAULT_VOXEL_BUDGET if budget is None else budget)
        self._conf = conf
        h = _lib.load().fvv_frame_create(_lib.host_ptr(self._tab), ctypes.c_int(self.ncam),
                                         _lib.host_ptr(conf))
        if not h:
            raise ValueError(_lib.load().fvv_last_error().decode(errors="replace"))
        self._h = ctypes.c_void_p(h)
        self._ranks = {}

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                _lib.load().fvv_frame_destroy(h)
            except Exception:  # noqa: BLE001
                pass
            self._h = None

    def _virtual_args(self, virtual):
        """(fvv_camera record, rank positions) of a virtual camera and their
        pointers, memoised on its parameter values: cam_table returns the
        same record object for equal values, so a camera mutated in place
        between frames gets a fresh ranking."""
        from .render import rank_cameras

        vt = cam_table([virtual])
        hit = self._ranks.get(id(vt))
        if hit is None or hit[0] is not vt:
            pos = {c.id: i for i, c in enumerate(self.cams)}
            arr = np.array([pos[i] for i in rank_cameras(virtual, self.cams)], dtype=np.int32)
            if len(self._ranks) > 64:
                self._ranks.clear()
            hit = (vt, arr, _lib.host_ptr(vt), _lib.host_ptr(arr))
            self._ranks[id(vt)] = hit
        return hit

    def _rank_pos(self, virtual):
        return self._virtual_args(virtual)[1]

    @property
    def stage_times(self) -> bool:
        return getattr(self, "_stage_times", True)

    @stage_times.setter
    def stage_times(self, on: bool) -> None:
        """Per-stage device times in each run's stats (ms); off saves ~22 us
        of host time per device-planned frame (fvv_frame_set_stage_times)."""
        _lib.load().fvv_frame_set_stage_times(self._h, ctypes.c_int(1 if on else 0))
        self._stage_times = bool(on)

    @property
    def last_mode(self) -> int:
        """How the last run went: 0 host-planned, 1 device-planned, 2 captured
        as a CUDA graph, 3 graph replay (fvv_frame_last_mode)."""
        return int(_lib.load().fvv_frame_last_mode(self._h))

    def run(self, masks, virtual=None, frames_buf=None, frame_off=None, fallback=None):
        """masks: uint8 (N,H,W) (or flat) CUDA tensor in rig order; for the
        colour pass, frames_buf (uint8 CUDA tensor, or the int base address of
        mapped pinned host frames, see fvv_host_mapped) + frame_off (int64
        byte offset of each camera's (H, W, 3) frame from that base)."""
        masks = mask_bytes(masks).reshape(-1)
        stats = np.zeros(1, dtype=_lib.FRAME_STATS_DTYPE)
        stage = ctypes.c_int(0)
        if virtual is not None:
            if frames_buf is None:
                raise ValueError("the colour pass needs frames_buf/frame_off")
            _, _, vt_p, rank_p = self._virtual_args(virtual)
            fb_p = _fallback_ptr() if fallback is None else _lib.host_ptr(np.ascontiguousarray(
                np.asarray(fallback, dtype=np.uint8).reshape(3)))
            fptr = ctypes.c_void_p(int(frames_buf)) if isinstance(frames_buf, int) else \
                _lib.dev_ptr(frames_buf)
            args = (vt_p, rank_p, fptr,
                    _lib.host_ptr(np.ascontiguousarray(frame_off, dtype=np.int64)), fb_p)
        else:
            args = (ctypes.c_void_p(0),) * 5
        rc = _lib.load().fvv_frame_run(self._h, _lib.dev_ptr(masks), *args, stream_handle(),
                                       _lib.host_ptr(stats), ctypes.byref(stage))
        if rc != 0:
            from .pipeline import StageError

            msg = _lib.load().fvv_last_error().decode(errors="replace")
            cause = ValueError(msg) if rc in (_lib.FVV_E_ARG, _lib.FVV_E_LIMIT) else \
                _lib.FvvError(msg)
            raise StageError(STAGE_NAMES.get(stage.value, "B-1 sparse carve"), cause)
        outs = _lib.FrameOutputs()
        _lib.load().fvv_frame_get_outputs(self._h, ctypes.byref(outs))
        n = int(outs.n_rois)  # (fvv_frame_get_rois writes all n entries)
        cid = np.empty(max(n, 1), dtype=np.int64)
        boxes = np.empty((max(n, 1), 6))
        grids = np.empty(max(n, 1), dtype=_lib.GRID_DTYPE)
        info = np.empty((max(n, 1), 8), dtype=np.int64)
        _lib.load().fvv_frame_get_rois(self._h, _lib.host_ptr(cid), _lib.host_ptr(boxes),
                                       _lib.host_ptr(grids), _lib.host_ptr(info))
        return FrameOutput(stats[0], outs, (cid[:n], boxes[:n], grids[:n], info[:n]),
                           self.ncam, virtual, self._h, owner=self)


_EXECUTORS = OrderedDict()
_MAX_EXECUTORS = 32


def executor_for(cfg, rig, slot: int = 0) -> FrameExecutor:
    """Executors are cached per (config, rig parameters, slot) so repeated
    run_frame / run_sequence calls reuse the device buffers; run_sequence
    gives each lane two slots, so one frame's D2H overlaps the lane's next
    frame."""
    from dataclasses import astuple

    key = (astuple(cfg), cam_table(list(rig)).tobytes(), int(slot))
    ex = _EXECUTORS.get(key)
    if ex is None:
        while len(_EXECUTORS) >= _MAX_EXECUTORS:
            # least recently used first; a FrameOutput still holding the
            # evicted executor keeps its buffers alive until it is dropped
            _EXECUTORS.popitem(last=False)
        ex = FrameExecutor(cfg, rig)
        _EXECUTORS[key] = ex
    else:
        _EXECUTORS.move_to_end(key)
    return ex


# ---------------------------------------------------------------- native sequences
class _SeqOwner:
    """Frees a native sequence result (its pinned block and device payload)
    when the last array or tensor viewing it is gone."""

    __slots__ = ("h",)

    def __init__(self, h):
        self.h = h

    def __del__(self):
        if self.h:
            try:
                _lib.load().fvv_seq_result_free(ctypes.c_void_p(self.h))
            except Exception:  # noqa: BLE001  (interpreter shutdown)
                pass
            self.h = None


_STATS_KEYS = ("sparse_tests", "sparse_occupied", "components", "dense_tests", "dense_occupied",
               "fallback_edges", "inconsistent_edge_starts", "triangles", "vertices", "n_rois",
               "covered_px", "sourced_px")


class SeqOutput:
    """One native-sequence frame: the FrameOutput fields the bundle builders
    read (stats, per-ROI tables, sizes), host arrays in the result's pinned
    block (views that keep it alive), and the device export payload."""

    def __init__(self, info, ncam, virtual, owner, frames):
        st = info.stats
        self.stats_raw = {k: int(getattr(st, k)) for k in _STATS_KEYS}
        self.stats_raw["ms"] = np.array(list(st.ms), dtype=np.float32)
        self.frame_id = int(info.id)
        self.ncam, self.virtual, self.frames = ncam, virtual, frames
        self.nv, self.nt = int(info.nv), int(st.triangles)
        self.vis_stride = int(info.vis_stride)
        n = int(info.n_rois)

        def arr(ptr, dtype, shape):
            if n == 0 or not ptr:
                return np.zeros(shape, dtype=dtype)
            nbytes = int(np.prod(shape)) * np.dtype(dtype).itemsize
            raw = (ctypes.c_uint8 * nbytes).from_address(ptr)
            return np.frombuffer(bytes(raw), dtype=dtype).reshape(shape)  # small: copied

        self.component_ids = arr(info.component_ids, np.int64, (n,))
        self.boxes = arr(info.boxes, np.float64, (n, 6))
        self.grids = arr(info.grids, _lib.GRID_DTYPE, (n,))
        self.info = arr(info.roi_info, np.int64, (n, 8))
        lay = np.array(list(info.layout), dtype=np.int64)
        self.layout = lay
        self.nbytes = int(lay[8:15].sum())
        self.host = {}
        total = int(lay[7])
        if info.host and total:
            carr = (ctypes.c_uint8 * total).from_address(info.host)
            carr._owner = owner  # numpy views -> memoryview -> carr -> owner
            raw = np.ctypeslib.as_array(carr)
            shapes = {"verts": ((self.nv, 3), np.float64), "tris": ((self.nt, 3), np.int32),
                      "vis": ((ncam, self.vis_stride), np.uint32)}
            if virtual is not None:
                h, w = virtual.image_height, virtual.image_width
                shapes.update(color=((h, w, 3), np.uint8), code=((h, w), np.int8))
            for i, name in enumerate(("verts", "tris", "vis", "color", "code")):
                off, nb = int(lay[i]), int(lay[8 + i])
                if name in shapes and (nb or name in ("verts", "tris", "vis")) and \
                        nb == int(np.prod(shapes[name][0])) * np.dtype(shapes[name][1]).itemsize:
                    shape, dt = shapes[name]
                    self.host[name] = raw[off:off + nb].view(dt).reshape(shape)
        self.payload = None
        if info.payload_dev:
            view = _CudaView(info.payload_dev, (max(int(info.payload_bytes), 1),), "|u1")
            view._owner = owner
            self.payload = torch.as_tensor(view, device="cuda")
        self._owner = owner

    def stats(self) -> dict:
        s = self.stats_raw
        return {k: int(s[k]) for k in _STATS_KEYS[:8]}


class NativeSequence:
    """fvv_seq (csrc/seq.cu): lanes of native threads, each with its own
    CUDA streams and two frame executors, run a video sequence frame by
    frame; submit() queues a frame, next() returns finished frames in
    submission order. The caller's interpreter lock is never held per frame
    on the lanes."""

    def __init__(self, cfg, rig, lanes=4, virtual=None, fallback=None, export=False):
        from .render import FALLBACK_COLOR, rank_cameras
        from .voxels import DEFAULT_VOXEL_BUDGET

        require_cuda()
        self.cams = list(rig)
        self.ncam = len(self.cams)
        self.virtual = virtual
        self.lanes = int(lanes)
        self._tab = cam_table(self.cams)
        conf = frame_config(cfg, DEFAULT_VOXEL_BUDGET)
        sc = _lib.SeqConfig()
        sc.lanes = self.lanes
        sc.readback_flags = 2 if virtual is not None else 0
        sc.has_virtual = int(virtual is not None)
        sc.export_payload = int(bool(export))
        if virtual is not None:
            ctypes.memmove(sc.virt, cam_table([virtual]).tobytes(), 192)
            pos = {c.id: i for i, c in enumerate(self.cams)}
            for r, cid in enumerate(rank_cameras(virtual, self.cams)):
                sc.rank_pos[r] = pos[cid]
        fb = np.asarray(FALLBACK_COLOR if fallback is None else fallback, dtype=np.uint8)
        for k in range(3):
            sc.fallback[k] = int(fb.reshape(3)[k])
        self._sc = sc
        self._mask_px = [c.image_height * c.image_width for c in self.cams]
        lib = _lib.load()
        h = lib.fvv_seq_create(_lib.host_ptr(self._tab), ctypes.c_int(self.ncam),
                               _lib.host_ptr(conf), ctypes.byref(sc))
        if not h:
            raise ValueError(lib.fvv_last_error().decode(errors="replace"))
        self._h = ctypes.c_void_p(h)
        self._pending = {}
        self.h2d_masks = 0  # silhouette bytes uploaded
        self.h2d_frames = 0  # colour bytes over PCIe (zero-copy taps or uploads)

    def close(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            lib = _lib.load()
            while True:  # results never collected: free them
                res = ctypes.c_void_p()
                if lib.fvv_seq_next(h, 1, ctypes.byref(res)) != 1:
                    break
                lib.fvv_seq_result_free(res)
            lib.fvv_seq_destroy(h)
            self._h = None
            self._pending.clear()

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass

    @staticmethod
    def _piece(a, keep):
        if isinstance(a, torch.Tensor):
            a = mask_bytes(a) if a.dtype != torch.uint8 else a
            a = a.contiguous()
            keep.append(a)
            return a.data_ptr(), a.numel() * a.element_size(), a.is_cuda
        arr = np.asarray(a)
        if arr.dtype == np.bool_:
            arr = arr.view(np.uint8)
        elif arr.dtype != np.uint8:
            arr = (arr != 0).view(np.uint8)
        arr = np.ascontiguousarray(arr)
        keep.append(arr)
        return arr.ctypes.data, arr.size, False

    def submit(self, frame_id, sils, frames=None):
        """Queue one frame: ``sils`` in rig order (list of (H, W) arrays or
        tensors, a stacked (N, H, W) or flat tensor, or a dict by camera
        id); ``frames`` a dict camera id -> (H, W, 3) uint8 for the colour
        pass. Inputs must stay unmodified until the frame is returned."""
        keep = []
        if isinstance(sils, torch.Tensor) and sils.dim() in (1, 3):
            pieces = [self._piece(sils.reshape(-1), keep)]
        else:
            sl = [sils[c.id] for c in self.cams] if isinstance(sils, dict) else list(sils)
            if len(sl) != self.ncam:
                raise ValueError(f"{len(sl)} silhouettes for {self.ncam} cameras")
            pieces = []
            for c, sv in zip(self.cams, sl):
                shp = tuple(sv.shape)
                if shp != (c.image_height, c.image_width):
                    raise ValueError(f"camera {c.id}: silhouette shape {shp} != "
                                     f"({c.image_height}, {c.image_width})")
                pieces.append(self._piece(sv, keep))
        if sum(n for _, n, _ in pieces) != sum(self._mask_px):
            raise ValueError("silhouettes do not match the rig's image sizes")
        ptrs = np.array([p for p, _, _ in pieces], dtype=np.uint64)
        sizes = np.array([n for _, n, _ in pieces], dtype=np.int64)
        fptr = None
        zero_copy = False
        if self.virtual is not None and frames is not None:
            fp = []
            for c in self.cams:
                f = frames[c.id]
                p, n, acc = self._piece(f, keep)
                if n != 3 * c.image_height * c.image_width:
                    raise ValueError(f"camera {c.id}: colour frame has {n} bytes")
                fp.append(p)
            fptr = np.array(fp, dtype=np.uint64)
            zero_copy = all(isinstance(frames[c.id], torch.Tensor) and
                            (frames[c.id].is_cuda or frames[c.id].is_pinned()) for c in self.cams)
        in_place = len(pieces) == 1 and isinstance(keep[0], torch.Tensor) and keep[0].is_cuda
        keep += [ptrs, sizes]
        self._pending[int(frame_id)] = (keep, frames, zero_copy, not in_place)
        rc = _lib.load().fvv_seq_submit(
            self._h, ctypes.c_int64(int(frame_id)), ctypes.c_void_p(ptrs.ctypes.data),
            ctypes.c_void_p(sizes.ctypes.data), ctypes.c_int(len(pieces)),
            ctypes.c_void_p(fptr.ctypes.data) if fptr is not None else None)
        if rc != 0:
            self._pending.pop(int(frame_id), None)
            raise ValueError(_lib.load().fvv_last_error().decode(errors="replace"))

    def next(self, wait=True):
        """The next finished frame (SeqOutput) in submission order, or None."""
        from .pipeline import StageError

        lib = _lib.load()
        res = ctypes.c_void_p()
        if lib.fvv_seq_next(self._h, int(bool(wait)), ctypes.byref(res)) != 1:
            return None
        owner = _SeqOwner(res.value)
        info = _lib.SeqResultInfo()
        lib.fvv_seq_result_get(res, ctypes.byref(info))
        keep, frames, zero_copy, uploaded_masks = self._pending.pop(int(info.id), (None,) * 4)
        if info.status != 0:
            msg = (info.err or b"").decode(errors="replace")
            cause = ValueError(msg) if info.status in (_lib.FVV_E_ARG, _lib.FVV_E_LIMIT) else \
                _lib.FvvError(msg)
            raise StageError(STAGE_NAMES.get(int(info.stage), "B-1 sparse carve"), cause)
        out = SeqOutput(info, self.ncam, self.virtual, owner, frames)
        if uploaded_masks:
            self.h2d_masks += sum(self._mask_px)
        if self.virtual is not None and frames is not None:
            self.h2d_frames += (12 * out.stats_raw["sourced_px"] if zero_copy else
                                3 * sum(self._mask_px))
        return out


_SEQUENCES = OrderedDict()


def sequence_for(cfg, rig, lanes, virtual, fallback, export=False) -> NativeSequence:
    """Native sequences are cached per (config, rig, lanes, view, fallback,
    export) and reused by later run_sequence calls."""
    from dataclasses import astuple

    key = (astuple(cfg), cam_table(list(rig)).tobytes(), int(lanes),
           None if virtual is None else cam_table([virtual]).tobytes(),
           None if fallback is None else tuple(int(v) for v in np.asarray(fallback).reshape(-1)),
           bool(export))
    seq = _SEQUENCES.get(key)
    if seq is None:
        while len(_SEQUENCES) >= 4:
            _SEQUENCES.popitem(last=False)[1].close()
        seq = NativeSequence(cfg, rig, lanes, virtual, fallback, export)
        _SEQUENCES[key] = seq
    else:
        _SEQUENCES.move_to_end(key)
    return seq


def _close_sequences():
    while _SEQUENCES:
        _SEQUENCES.popitem()[1].close()


import atexit  # noqa: E402

atexit.register(_close_sequences)
