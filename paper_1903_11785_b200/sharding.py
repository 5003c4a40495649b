"""Frame sharding across GPUs.

Frames are independent (pipeline.py:115-220 keeps no cross-frame state), so
N processes (one per GPU, torchrun) split a sequence by frame index with no
collective on the data path. The helpers here are the whole multi-GPU layer:
frame assignment, the max-over-ranks timer reduction the benchmark uses,
and the optional gather of finished per-frame results to rank 0 (for the
bundle writer; outside the timed hot path).
"""

from __future__ import annotations

import os


def world():
    """(rank, world_size, local_rank) from the torchrun environment."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def frames_for_rank(rank: int, world_size: int, n_frames: int) -> list:
    """Round-robin: frame f -> rank f mod N (balanced to within one frame)."""
    if not (0 <= rank < world_size):
        raise ValueError(f"rank {rank} outside world of {world_size}")
    return list(range(rank, n_frames, world_size))


def reduce_max(value: float, group=None) -> float:
    """Max over ranks (device timers: the slowest rank defines the job time)."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return float(value)
    dev = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
    t = torch.tensor([float(value)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def reduce_sum(value: float, group=None) -> float:
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return float(value)
    dev = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
    t = torch.tensor([float(value)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return float(t.item())


def gather_to_rank0(items: dict, group=None):
    """Gather {frame_id: payload} dicts (e.g. mesh arrays + visibility bits)
    from every rank to rank 0; returns the merged dict on rank 0, None
    elsewhere. Host objects, so it works over gloo and nccl alike."""
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return dict(items)
    out = [None] * dist.get_world_size(group) if dist.get_rank(group) == 0 else None
    dist.gather_object(items, out, dst=0, group=group)
    if out is None:
        return None
    merged = {}
    for part in out:
        merged.update(part)
    return dict(sorted(merged.items()))


# ---------------------------------------------------------------- frame export
# A finished frame's mesh + visibility in one byte payload (device or host
# memory) plus a float64 meta vector: what a frame-sharded rank sends to
# rank 0, whose bundle writer (bundle.py, reference bundle.py:77-136)
# consumes it. Meta layout (every entry an integer < 2^53 or a time in ms):
#   [0] _MAGIC [1] nv [2] nt [3] ncam [4] vis_stride [5] nroi
#   [6:14] stats (sparse_tests .. triangles) [14:20] stage ms (B-1 .. D-2)
#   [20:20+nroi] component ids, then nroi x 8 per-ROI mesh info
#   (vertex base, vertices, cell base, cells, triangle base, triangles,
#   fallback edges, inconsistent starts).
_MAGIC = 1903.11785
_STATS = ("sparse_tests", "sparse_occupied", "components", "dense_tests", "dense_occupied",
          "fallback_edges", "inconsistent_edge_starts", "triangles")
_HDR = 20
GATHER_BYTES = {"payload": 0}  # payload bytes rank 0 received (and read back)


def payload_layout(nv, nt, ncam, vis_stride):
    """Byte (offset, size) of vertices (f64 nv x 3), triangles (i32 nt x 3)
    and visibility bits (u32 ncam x vis_stride) in a payload, 256-aligned."""
    sizes = (24 * int(nv), 12 * int(nt), 4 * int(ncam) * int(vis_stride))
    offs, o = [], 0
    for n in sizes:
        offs.append((o, n))
        o += (n + 255) & ~255
    return offs, o


def export_meta(stats, ms, component_ids, info, nv, nt, ncam, vis_stride):
    import numpy as np

    nroi = len(component_ids)
    meta = np.zeros(_HDR + 9 * nroi, dtype=np.float64)
    meta[:6] = (_MAGIC, nv, nt, ncam, vis_stride, nroi)
    meta[6:14] = [float(stats[k]) for k in _STATS]
    meta[14:20] = np.asarray(ms, dtype=np.float64)[:6]
    meta[_HDR:_HDR + nroi] = np.asarray(component_ids, dtype=np.float64)
    meta[_HDR + nroi:] = np.asarray(info, dtype=np.float64).reshape(-1)
    return meta


def export_from_arrays(stats, ms, component_ids, info, verts, tris, vis_bits):
    """Host-side export (meta, uint8 payload tensor) from numpy arrays: the
    same format FrameOutput.export writes on the device."""
    import numpy as np
    import torch

    verts = np.ascontiguousarray(verts, dtype=np.float64).reshape(-1, 3)
    tris = np.ascontiguousarray(tris, dtype=np.int32).reshape(-1, 3)
    vis_bits = np.ascontiguousarray(vis_bits, dtype=np.uint32)
    ncam, stride = vis_bits.shape
    meta = export_meta(stats, ms, component_ids, info, len(verts), len(tris), ncam, stride)
    offs, total = payload_layout(len(verts), len(tris), ncam, stride)
    buf = np.zeros(max(total, 1), dtype=np.uint8)
    for (off, n), a in zip(offs, (verts, tris, vis_bits)):
        buf[off:off + n] = a.reshape(-1).view(np.uint8)
    return meta, torch.from_numpy(buf)


class _ExportedOutput:
    """The parts of an executor FrameOutput that pipeline.bundle_from_output
    reads, rebuilt from an export's meta vector."""

    def __init__(self, meta):
        import numpy as np

        if meta[0] != _MAGIC:
            raise ValueError("not a frame export")
        self.nv, self.nt, self.ncam, self.vis_stride, nroi = (int(v) for v in meta[1:6])
        self._stats = {k: int(v) for k, v in zip(_STATS, meta[6:14])}
        self.stats_raw = {"ms": np.asarray(meta[14:20], dtype=np.float32)}
        self.component_ids = meta[_HDR:_HDR + nroi].astype(np.int64)
        self.info = meta[_HDR + nroi:].astype(np.int64).reshape(nroi, 8)

    def stats(self):
        return dict(self._stats)


def bundle_from_export(meta, payload_host, cfg, rig, frame_id, frames=None):
    """SceneBundle of an exported frame (payload already on the host)."""
    import numpy as np

    from .pipeline import bundle_from_output

    out = _ExportedOutput(meta)
    raw = payload_host.numpy() if hasattr(payload_host, "numpy") else np.asarray(payload_host)
    (ov, nvb), (ot, ntb), (ob, nbb) = payload_layout(out.nv, out.nt, out.ncam, out.vis_stride)[0]
    host = {"verts": raw[ov:ov + nvb].view(np.float64).reshape(out.nv, 3),
            "tris": raw[ot:ot + ntb].view(np.int32).reshape(out.nt, 3),
            "vis": raw[ob:ob + nbb].view(np.uint32).reshape(out.ncam, out.vis_stride)}
    return bundle_from_output(out, host, cfg, rig, frames, frame_id, keep_device=False)


# ---------------------------------------------------------------- gather
class FrameGather:
    """Point-to-point transport of frame exports to rank 0. The small meta
    vector travels over a gloo group (host memory); the payload over the data
    group: NCCL straight from the sender's device buffer into a device
    buffer on rank 0 (NVLink), or gloo with host tensors on CPU-only runs.
    Each sender sends its frames in ascending order and rank 0 posts its
    receives in ascending frame order, so every pair's messages match."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.data_group = group
        backend = dist.get_backend(group)
        self.nccl = backend == "nccl"
        # collective over all ranks: every rank constructs its FrameGather
        self.meta_group = dist.new_group(backend="gloo") if self.nccl else group
        self._streams = None
        self._inflight = []
        self._device = None
        if self.nccl:
            import torch

            self._device = torch.cuda.current_device()

    def _stream(self):
        import torch

        # the receiver runs on its own thread: CUDA's current device is per thread
        torch.cuda.set_device(self._device)
        if self._streams is None:
            self._streams = torch.cuda.Stream()
        return self._streams

    def send(self, meta, payload, ready_event=None, dst=0):
        import numpy as np
        import torch
        import torch.distributed as dist

        head = torch.tensor([len(meta), payload.numel()], dtype=torch.int64)
        dist.send(head, dst, group=self.meta_group)
        dist.send(torch.from_numpy(np.ascontiguousarray(meta)), dst, group=self.meta_group)
        if self.nccl:
            st = self._stream()
            with torch.cuda.stream(st):
                if ready_event is not None:
                    st.wait_event(ready_event)
                dist.send(payload, dst, group=self.data_group)
                done = torch.cuda.Event()
                done.record(st)
            # the payload may be a view of a native sequence result's device
            # block (not torch-allocated: record_stream cannot guard it):
            # hold it until its send has completed
            self._inflight.append((done, payload))
            while self._inflight and self._inflight[0][0].query():
                self._inflight.pop(0)
        else:
            dist.send(payload.cpu(), dst, group=self.data_group)

    def recv(self, src):
        """(meta, host payload, completion event or None) of src's next frame."""
        import torch
        import torch.distributed as dist

        head = torch.zeros(2, dtype=torch.int64)
        dist.recv(head, src, group=self.meta_group)
        meta = torch.zeros(int(head[0]), dtype=torch.float64)
        dist.recv(meta, src, group=self.meta_group)
        n = int(head[1])
        GATHER_BYTES["payload"] += n
        if not self.nccl:
            buf = torch.empty(n, dtype=torch.uint8)
            dist.recv(buf, src, group=self.data_group)
            return meta.numpy(), buf, None
        st = self._stream()
        with torch.cuda.stream(st):
            dbuf = torch.empty(n, dtype=torch.uint8, device="cuda")
            dist.recv(dbuf, src, group=self.data_group)
            host = torch.empty(n, dtype=torch.uint8, pin_memory=True)
            host.copy_(dbuf, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(st)
        return meta.numpy(), host, ev


def merge_sharded(rank, world, n_frames, local, gather, to_bundle):
    """The frame-sharded sequence protocol, independent of
    how frames are computed. ``local`` yields (frame_id, bundle, image,
    export) for this rank's frames (frames_for_rank order); ``gather`` is a
    FrameGather or None; ``to_bundle(frame_id, meta, payload, event)`` turns
    a received export into a SceneBundle. Ranks other than 0 send every
    export to rank 0 and yield (frame_id, None, image); rank 0 yields
    (frame_id, bundle, image or None) for EVERY frame of the sequence in
    frame order, receiving the other ranks' frames on a background thread
    while its own frames run."""
    import threading

    if world == 1 or gather is None:
        for fid, bundle, img, _ in local:
            yield fid, bundle, img
        return
    if rank != 0:
        for fid, _, img, exp in local:
            meta, payload, ev = exp
            gather.send(meta, payload, ev)
            yield fid, None, img
        return
    remote = [f for f in range(n_frames) if f % world != 0]
    got = {}
    cond = threading.Condition()
    failure = []

    def receiver():
        try:
            for f in remote:
                item = gather.recv(f % world)
                with cond:
                    got[f] = item
                    cond.notify_all()
        except BaseException as exc:  # noqa: BLE001  (re-raised on the caller's thread)
            with cond:
                failure.append(exc)
                cond.notify_all()

    th = threading.Thread(target=receiver, name="fvv-gather", daemon=True)
    th.start()
    local = iter(local)
    for f in range(n_frames):
        if f % world == 0:
            fid, bundle, img, _ = next(local)
            if fid != f:
                raise RuntimeError(f"rank 0 produced frame {fid}, expected {f}")
            yield f, bundle, img
            continue
        with cond:
            while f not in got and not failure:
                cond.wait()
            if failure:
                raise failure[0]
            meta, payload, ev = got.pop(f)
        yield f, to_bundle(f, meta, payload, ev), None
    th.join()


_GATHERS = {}


def frame_gather(group=None):
    """The FrameGather of a process group (created once: collective)."""
    key = id(group)
    g = _GATHERS.get(key)
    if g is None:
        g = _GATHERS[key] = FrameGather(group)
    return g
