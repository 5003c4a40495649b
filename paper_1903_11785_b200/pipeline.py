"""Per-frame orchestration on the GPU (drop-in for freeview.pipeline).

``run_frame`` keeps the reference's signature, stage names, stats and
errors (pipeline.py:34-220). Inside, every stage runs on the current CUDA
stream with its inputs resident on the device:

  B-1 fvv_carve (stage grid)      -> occupancy bits
  B-2 fvv_ccl26 -> component table (host sync #1: the ROI table is host
      bookkeeping, hull.py:272-284, computed with numpy like the reference)
  B-3 fvv_carve (all ROI grids in one launch)
  C   fvv_mesh_prepare / fvv_mesh_emit (host sync #2: output sizes)
  D-1 fvv_rasterize (all cameras in one launch; triangle count read on device)
  D-2 fvv_classify  (all cameras, visibility as bits)

Stage timings are CUDA-event device times. Host views (meshes, visibility
flags, depth images) are materialised when the bundle is read.
"""

from __future__ import annotations

import json
from dataclasses import asdict, dataclass, replace

import numpy as np
import torch

from ._device import DeviceSilhouettes, mask_bytes, require_cuda
from .bundle import SceneBundle, StageTimings
from .hull import NoiseFilterParams, Roi, carve_grids, finish_labels, label_grid_async
from .mesh import TriangleMesh, polygonize_grids
from .silhouette import AdaptiveParams, silhouettes_device
from .visibility import bits_to_flags, classify_bits, raster_planes
from .voxels import GridSpec


class StageError(RuntimeError):
    """A pipeline stage failed; ``stage`` names it (pipeline.py:34-38)."""

    def __init__(self, stage: str, cause: Exception):
        super().__init__(f"[{stage}] {cause}")
        self.stage = stage
        self.cause = cause


@dataclass
class PipelineConfig:
    """pipeline.py:41-101, same fields, defaults, validation and JSON form."""

    stage_lo: tuple = (-9000.0, -9000.0, 0.0)
    stage_hi: tuple = (9000.0, 9000.0, 9000.0)
    coarse_spacing: float = 50.0
    fine_spacing: float = 20.0
    min_views: int = 1
    t_small: int = 5
    t_large: float = float("inf")
    roi_margin: float = None  # default: one coarse voxel
    t_v: float = None  # default: 3 * fine_spacing
    iso_mode: str = "exact"
    fixed_isovalue: float = 0.5
    theta_near: float = 3.0
    theta_far: float = 8.0
    d_max: float = 32.0
    block_dims: tuple = (16, 16, 16)
    workers: int = 1

    def __post_init__(self) -> None:
        self.stage_lo = tuple(float(v) for v in self.stage_lo)
        self.stage_hi = tuple(float(v) for v in self.stage_hi)
        if self.fine_spacing > self.coarse_spacing:
            raise ValueError("fine_spacing must be <= coarse_spacing")
        if any(hi <= lo for lo, hi in zip(self.stage_lo, self.stage_hi)):
            raise ValueError("stage volume must be nonempty")
        if self.t_small < 0 or self.t_v is not None and self.t_v < 0:
            raise ValueError("thresholds must be nonnegative")
        if self.roi_margin is None:
            self.roi_margin = self.coarse_spacing
        if self.t_v is None:
            self.t_v = 3.0 * self.fine_spacing
        if self.iso_mode not in ("exact", "fixed"):
            raise ValueError(f"unknown isovalue mode {self.iso_mode!r}")

    @property
    def adaptive_params(self) -> AdaptiveParams:
        return AdaptiveParams(self.theta_near, self.theta_far, self.d_max)

    @property
    def noise_params(self) -> NoiseFilterParams:
        return NoiseFilterParams(self.t_small, self.t_large)

    def coarse_spec(self) -> GridSpec:
        return GridSpec.from_aabb(self.stage_lo, self.stage_hi, self.coarse_spacing)

    def to_json(self, path) -> None:
        d = asdict(self)
        d["t_large"] = None if np.isinf(self.t_large) else self.t_large
        with open(path, "w", encoding="utf-8") as fh:
            json.dump(d, fh, indent=2)
            fh.write("\n")

    @classmethod
    def from_json(cls, path) -> "PipelineConfig":
        with open(path, "r", encoding="utf-8") as fh:
            d = json.load(fh)
        if d.get("t_large") is None:
            d["t_large"] = float("inf")
        return cls(**{k: (tuple(v) if isinstance(v, list) else v) for k, v in d.items()})


class _StageClock:
    """CUDA events at stage boundaries on the current stream."""

    def __init__(self):
        self.marks = []

    def mark(self, name):
        ev = torch.cuda.Event(enable_timing=True)
        ev.record()
        self.marks.append((name, ev))

    def timings(self) -> StageTimings:
        t = StageTimings()
        for (_, a), (name, b) in zip(self.marks, self.marks[1:]):
            setattr(t, name, a.elapsed_time(b))
        return t


class FrameResult:
    """Device-side outputs of B-1 .. D-2 for one frame."""

    def __init__(self):
        self.stats = {}


def reconstruct(cfg: PipelineConfig, rig, dsils: DeviceSilhouettes, clock=None) -> FrameResult:
    """B-1 .. D-2 for one frame composed from the per-stage public functions
    (hull / mesh / visibility); outputs stay on the device. ``run_frame`` uses
    the native executor (executor.py) instead; tests check the two agree."""
    r = FrameResult()
    clock = clock or _StageClock()
    cams = list(rig)

    def stage(name, fn):
        try:
            return fn()
        except StageError:
            raise
        except Exception as exc:  # noqa: BLE001  (reference wraps every failure)
            raise StageError(name, exc) from exc

    spec = cfg.coarse_spec()
    r.spec = spec
    r.stats["sparse_tests"] = spec.num_voxels
    clock.mark("start")
    r.coarse = stage("B-1 sparse carve", lambda: carve_grids(dsils, [spec], cfg.min_views)[0])
    clock.mark("sparse_carve")

    def b2():
        lab = finish_labels(r.coarse, *label_grid_async(r.coarse))
        params = cfg.noise_params
        comps = [c for c in lab.components if params.keeps(c.voxel_count)]
        rois = []
        for c in comps:  # hull.py:272-284 with the reference's numpy expressions
            lo = spec.origin + spec.spacing * np.asarray(c.bbox_min, dtype=np.float64) - \
                cfg.roi_margin
            hi = spec.origin + spec.spacing * (np.asarray(c.bbox_max, dtype=np.float64) + 1.0) \
                + cfg.roi_margin
            rois.append(Roi(np.maximum(lo, spec.origin), np.minimum(hi, spec.extent), c.id))
        return lab, comps, rois

    r.labeling, r.components, r.rois = stage("B-2 noise filter/ROI", b2)
    r.stats["sparse_occupied"] = r.coarse.occupied_count  # synced by B-2 already
    r.stats["components"] = len(r.components)
    clock.mark("noise_filter_roi")

    def b3():
        specs = [GridSpec.from_aabb(roi.lo, roi.hi, cfg.fine_spacing) for roi in r.rois]
        return carve_grids(dsils, specs, cfg.min_views) if specs else []

    r.fine = stage("B-3 dense carve", b3)
    r.stats["dense_tests"] = sum(g.spec.num_voxels for g in r.fine)
    clock.mark("dense_carve")

    def c():
        if not r.fine:
            return None
        return polygonize_grids(r.fine, rig, dsils, cfg.iso_mode, cfg.fixed_isovalue,
                                [roi.component_id for roi in r.rois])

    r.batch = stage("C polygonize", c)
    clock.mark("polygonize")
    if r.batch is not None and r.batch.verts.shape[0] > 0:
        verts, tris = r.batch.verts, r.batch.tris
        nt_dev = r.batch.num_triangles_dev
        r.planes = stage("D-1 depth images",
                         lambda: raster_planes(verts, tris, cams, want_ids=False, nt_dev=nt_dev))
        clock.mark("depth_images")
        r.vis_bits = stage("D-2 visibility",
                           lambda: classify_bits(verts, tris, r.planes, cfg.t_v, nt_dev=nt_dev))
        clock.mark("visibility")
    else:
        r.planes = None
        r.vis_bits = None
        clock.mark("depth_images")
        clock.mark("visibility")
    r.clock = clock
    return r


def _finish_stats(r: FrameResult):
    """Read the device-side counts (one sync) into the reference's stats keys."""
    dense_counts = [g._count for g in r.fine]
    if getattr(r, "_dense_occ", None) is not None:
        r.stats["dense_occupied"] = int(r._dense_occ)
    elif dense_counts:
        occ = torch.stack([c.reshape(()) for c in dense_counts]).cpu().numpy()
        r.stats["dense_occupied"] = int(occ.sum())
    else:
        r.stats["dense_occupied"] = 0
    if r.batch is not None:
        totals, _ = r.batch.host_info()
        st = [r.batch.stats(g) for g in range(len(r.fine))]
        r.stats["fallback_edges"] = sum(s.fallback_edges for s in st)
        r.stats["inconsistent_edge_starts"] = sum(s.inconsistent_starts for s in st)
        r.stats["triangles"] = int(totals[2])
    else:
        r.stats["fallback_edges"] = 0
        r.stats["inconsistent_edge_starts"] = 0
        r.stats["triangles"] = 0


class _LazyVisibility(dict):
    """camera id -> (T,) bool, unpacked from the device bit rows on first read."""

    def __init__(self, ids, bits_host, n):
        super().__init__()
        self._ids = list(ids)
        self._bits = bits_host
        self._n = n
        for i in self._ids:
            dict.__setitem__(self, i, None)

    def __getitem__(self, key):
        v = dict.__getitem__(self, key)
        if v is None:
            row = self._ids.index(key)
            v = bits_to_flags(self._bits[row], self._n) if self._n else np.zeros(0, dtype=bool)
            dict.__setitem__(self, key, v)
        return v

    def values(self):
        return [self[k] for k in self._ids]

    def items(self):
        return [(k, self[k]) for k in self._ids]

    def get(self, key, default=None):
        return self[key] if key in self else default


def compute_silhouettes(cfg, rig, frames, proposals, background):
    """Adaptive silhouette extraction for every camera (pipeline.py:104-112),
    on the GPU (silhouette.py kernels); returns the reference's list of
    (H, W) bool masks in rig order."""
    masks = silhouettes_device(rig, frames, proposals, background, cfg.adaptive_params).cpu()
    out, off = [], 0
    for cam in rig:
        n = cam.image_height * cam.image_width
        out.append(masks[off:off + n].numpy().astype(bool).reshape(cam.image_height,
                                                                   cam.image_width))
        off += n
    return out


def _masks_on_device(rig, sils):
    """Validate like hull.py:63-75 (_check_sils) and return the masks as one
    uint8 CUDA tensor in rig order."""
    dev = require_cuda()
    cams = list(rig)
    if isinstance(sils, DeviceSilhouettes):
        if sils.ncam != len(cams):
            raise ValueError(f"{sils.ncam} silhouettes for {len(cams)} cameras")
        return sils._masks
    if isinstance(sils, torch.Tensor) and sils.dim() == 1:  # flat, rig order (internal)
        if sils.numel() != sum(c.image_height * c.image_width for c in cams):
            raise ValueError("flat silhouette buffer does not match the rig's image sizes")
        return mask_bytes(sils).to(dev, non_blocking=True)
    if len(sils) != len(cams):
        raise ValueError(f"{len(sils)} silhouettes for {len(cams)} cameras")
    if isinstance(sils, torch.Tensor) and sils.dim() == 3:
        shape = tuple(sils.shape[1:])
        for c in cams:
            if shape != (c.image_height, c.image_width):
                raise ValueError(f"camera {c.id}: silhouette shape {shape} != "
                                 f"({c.image_height}, {c.image_width})")
        return mask_bytes(sils).to(dev, non_blocking=True).reshape(-1)
    parts = []
    for c, s in zip(cams, sils):
        if isinstance(s, torch.Tensor):
            s = s.cpu().numpy()
        s = np.asarray(s)
        if s.shape != (c.image_height, c.image_width):
            raise ValueError(f"camera {c.id}: silhouette shape {s.shape} != "
                             f"({c.image_height}, {c.image_width})")
        parts.append(np.ascontiguousarray(s if s.dtype == np.bool_ else s.astype(bool)))
    out = torch.empty(sum(p.size for p in parts), dtype=torch.uint8, device=dev)
    o = 0
    for p in parts:
        out[o:o + p.size].copy_(torch.from_numpy(p.reshape(-1).view(np.uint8)))
        o += p.size
    return out


def bundle_from_output(out, host, cfg, rig, frames, frame_id=0, keep_depths=False,
                       keep_device=True) -> SceneBundle:
    """SceneBundle (bundle.py:55-74) from an executor run and its host copies."""
    cams = list(rig)
    stats = out.stats()
    t = StageTimings()
    for name, ms in zip(("sparse_carve", "noise_filter_roi", "dense_carve", "polygonize",
                         "depth_images", "visibility"), out.stats_raw["ms"][:6]):
        setattr(t, name, float(ms))
    verts, tris = host["verts"], host["tris"]
    meshes = []
    for g, cid in enumerate(out.component_ids):
        vb, nv, tb, nt = (int(out.info[g][k]) for k in (0, 1, 4, 5))
        if nv == 0:
            meshes.append(TriangleMesh.empty())
            continue

        def load(vb=vb, nv=nv, tb=tb, nt=nt, cid=cid):  # per-ROI views, built on access
            return (verts[vb:vb + nv], tris[tb:tb + nt] - np.int32(vb),
                    np.full(nt, int(cid), dtype=np.int32))

        meshes.append(TriangleMesh._lazy(nt, load))
    info = out.info
    if len(info) == 0 or np.all((info[:, 1] == 0) | (info[:, 5] > 0)):
        cids, counts = out.component_ids.astype(np.int32), info[:, 5].copy()

        def oids(cids=cids, counts=counts):  # built on first access
            return np.repeat(cids, counts) if len(counts) else np.zeros(0, dtype=np.int32)

        merged = TriangleMesh._trusted(verts if len(tris) else np.zeros((0, 3)), tris, oids)
    else:
        merged = TriangleMesh.concatenate(meshes)
    nt = stats["triangles"]
    vis = _LazyVisibility([c.id for c in cams], host["vis"], nt)
    if keep_device and nt and len(merged.vertices) == out.nv:
        merged._dev = (out.verts.clone(), out.tris.clone())
        vis._device_bits = out.vis_bits.clone()
    depths = {}
    if keep_depths:
        off = 0
        for c in cams:
            n = c.image_height * c.image_width
            depths[c.id] = (host["depth"][off:off + n].reshape(c.image_height, c.image_width)
                            if "depth" in host else
                            np.full((c.image_height, c.image_width), np.inf))
            off += n
    bundle = SceneBundle(frame_id=frame_id, rig=rig, meshes=meshes,
                         textures=dict(frames) if frames is not None else {}, visibility=vis,
                         timings=t, stats=stats, stage_lo=np.array(cfg.stage_lo),
                         stage_hi=np.array(cfg.stage_hi), depths=depths)
    bundle._merged = merged
    return bundle


def run_frame(cfg: PipelineConfig, rig, frames: dict, sils=None, proposals: dict = None,
              background: dict = None, frame_id: int = 0, keep_depths: bool = False) -> SceneBundle:
    """Reconstruct one frame into a SceneBundle (pipeline.py:115-220) on the GPU.

    Runs the native executor (csrc/frame.cu) for B-1 .. D-2 with the same
    stage names, stats and errors as the reference. ``sils`` may be the
    reference's list of (H, W) bool arrays, a stacked (N, H, W) uint8/bool
    tensor (pinned host or CUDA) or a DeviceSilhouettes."""
    if sils is None:
        if proposals is None or background is None:
            raise StageError("silhouette", ValueError("need sils or proposals+background"))
        try:  # silhouettes stay on the GPU (flat, rig order) and feed the carve
            sils = silhouettes_device(rig, frames, proposals, background, cfg.adaptive_params)
        except Exception as exc:
            raise StageError("silhouette", exc) from exc
    from .executor import executor_for

    cfg.coarse_spec()  # pipeline.py:151 validates the stage grid outside any stage
    try:
        masks = _masks_on_device(rig, sils)
        ex = executor_for(cfg, rig)
    except StageError:
        raise
    except Exception as exc:
        raise StageError("B-1 sparse carve", exc) from exc
    out = ex.run(masks)
    host = out.to_host(list(rig), keep_depths)
    return bundle_from_output(out, host, cfg, rig, frames, frame_id, keep_depths)


def bundle_from(r: FrameResult, cfg, rig, frames, frame_id=0, keep_depths=False) -> SceneBundle:
    """Host-side SceneBundle over a device FrameResult (one sync)."""
    _finish_stats(r)
    timings = r.clock.timings()
    cams = list(rig)
    meshes = r.batch.meshes() if r.batch is not None else []
    nt = r.stats["triangles"]
    if r.vis_bits is not None:
        vbits = r._vis_host if getattr(r, "_vis_host", None) is not None else \
            r.vis_bits.cpu().numpy()
        vis = _LazyVisibility([c.id for c in cams], vbits, nt)
        vis._device_bits = r.vis_bits  # render_view reads these directly (rig order)
    else:
        vis = {c.id: np.zeros(0, dtype=bool) for c in cams}
    depths = {}
    if keep_depths:
        for i, c in enumerate(cams):
            depths[c.id] = (r.planes.depth_of(i).cpu().numpy() if r.planes is not None
                            else np.full((c.image_height, c.image_width), np.inf))
    stats = {k: r.stats[k] for k in ("sparse_tests", "sparse_occupied", "components", "dense_tests",
                                     "dense_occupied", "fallback_edges",
                                     "inconsistent_edge_starts", "triangles")}
    bundle = SceneBundle(frame_id=frame_id, rig=rig, meshes=meshes,
                         textures=dict(frames) if frames is not None else {}, visibility=vis,
                         timings=timings, stats=stats, stage_lo=np.array(cfg.stage_lo),
                         stage_hi=np.array(cfg.stage_hi), depths=depths)
    bundle._merged = r.batch.merged() if r.batch is not None else TriangleMesh.empty()
    bundle._result = r
    return bundle


def _readback(r, image):
    """Copy every host-facing result of a frame back with two syncs: the
    small counters first (they size the rest), then the mesh, visibility
    bits and rendered image in one batch of async copies."""
    small = [torch.zeros(1, dtype=torch.int64, device=r.coarse.device_bits().device)]
    if r.fine:
        small.append(torch.stack([g._count.reshape(()) for g in r.fine]))
    if r.batch is not None:
        small += [r.batch._totals, r.batch._info.reshape(-1)]
    host = torch.cat(small).cpu().numpy()
    nf = len(r.fine)
    r._dense_occ = int(host[1:1 + nf].sum())
    if r.batch is None:
        return None
    totals = host[1 + nf:4 + nf].copy()
    info = host[4 + nf:].reshape(len(r.fine), 8).copy()
    r.batch._host = (totals, info)
    nt = int(totals[2])
    pinned = []

    def fetch(t):
        h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
        h.copy_(t, non_blocking=True)
        pinned.append(h)
        return h

    hv, ht = fetch(r.batch.verts), fetch(r.batch.tris[:nt])
    hb = fetch(r.vis_bits) if r.vis_bits is not None else None
    himg = [fetch(x) for x in image] if image is not None else None
    torch.cuda.current_stream().synchronize()
    r.batch._host_arrays = (hv.numpy(), ht.numpy())
    r._vis_host = hb.numpy() if hb is not None else None
    return [x.numpy() for x in himg] if himg is not None else None


def run_sequence(cfg: PipelineConfig, rig, frames_seq, sils_seq, virtual=None,
                 fallback_color=None, frame_id0: int = 0, lanes: int = 4):
    """Reconstruct (and, given ``virtual``, colour) a sequence of frames.

    The production form of run_frame + render_view for video, pipelined over
    CPU threads like the paper's system: the native sequence
    runner (csrc/seq.cu) sends frame f to lane f mod ``lanes``, a C++ thread
    with its own CUDA streams and two frame executors, which uploads the
    silhouettes, runs the frame and reads its results back into a pooled
    pinned block, so one lane's host synchronisations and small kernels
    overlap the other lanes' work and no Python runs per frame on the lanes
    (pinned colour frames are sampled in place by the colour pass). The
    caller's thread only queues inputs and turns finished frames into
    SceneBundles. Inputs should be pinned
    host tensors for the copies to be asynchronous; pinned colour frames are
    read in place by the GPU, so a frame's inputs must stay unmodified until
    that frame has been yielded (up to 2 x lanes frames are in flight).
    Yields (SceneBundle, RenderedImage or None) per frame, in input order,
    with the mesh, visibility flags and rendered image on the host."""
    for _, bundle, img, _ in _run_local(cfg, rig, frames_seq, sils_seq, virtual,
                                        fallback_color, _count_from(frame_id0), lanes):
        yield bundle, img


def _count_from(n):
    while True:
        yield n
        n += 1


def _run_local(cfg, rig, frames_seq, sils_seq, virtual, fallback_color, frame_ids, lanes,
               export=False):
    """run_sequence's engine over the native sequence runner (executor.
    NativeSequence, csrc/seq.cu). Yields (frame_id, SceneBundle or None,
    image or None, export or None) in input order. With ``export`` (a
    frame-sharded rank other than 0) the mesh and visibility bits are not
    read back: the lanes copy each frame's into a device payload
    (sharding.py format) for the caller to send to rank 0, and the bundle is
    None."""
    from .executor import sequence_for
    from .render import D2H_BYTES, H2D_BYTES, CodedImage

    require_cuda()
    lanes = max(1, int(lanes))
    cams = list(rig)
    rig_ids = [c.id for c in cams]
    seq = sequence_for(cfg, rig, lanes, virtual, fallback_color, export)
    caller = torch.cuda.current_stream()
    caller.synchronize()  # inputs the caller produced on its stream are complete
    fids = iter(frame_ids)
    h2d0 = (seq.h2d_masks, seq.h2d_frames)

    def finish(out):
        D2H_BYTES["results"] += out.nbytes
        host = out.host
        bundle = None if export else bundle_from_output(out, host, cfg, rig, out.frames,
                                                        out.frame_id, keep_device=False)
        img = CodedImage(host["color"], host["code"], rig_ids) if virtual is not None else None
        exp = None
        if export:
            from .sharding import export_meta

            meta = export_meta(out.stats(), out.stats_raw["ms"][:6], out.component_ids,
                               out.info, out.nv, out.nt, out.ncam, out.vis_stride)
            exp = (meta, out.payload, None)
        return out.frame_id, bundle, img, exp

    n_in = n_out = 0
    try:
        for frames, sils in zip(frames_seq, sils_seq):
            seq.submit(next(fids), sils, frames if virtual is not None else None)
            n_in += 1
            while n_out < n_in:  # hand back, in order, every frame already done
                out = seq.next(wait=n_in - n_out > 2 * lanes)  # bound the frames in flight
                if out is None:
                    break
                n_out += 1
                yield finish(out)
        while n_out < n_in:
            out = seq.next(wait=True)
            n_out += 1
            yield finish(out)
    finally:
        while n_out < n_in:  # closed early or failed: drain (results free themselves)
            try:
                if seq.next(wait=True) is None:
                    break
            except Exception:  # noqa: BLE001
                pass
            n_out += 1
        H2D_BYTES["masks"] += seq.h2d_masks - h2d0[0]
        H2D_BYTES["frames"] += seq.h2d_frames - h2d0[1]


def run_sequence_sharded(cfg: PipelineConfig, rig, source, n_frames: int, virtual=None,
                         fallback_color=None, lanes: int = 4, gather: bool = True, group=None):
    """run_sequence over a frame-sharded job: one process per GPU
    (torch.distributed initialised, NCCL), frame f on rank f mod N
    (frames are independent, pipeline.py:115-220).

    ``source(f) -> (frames, sils)`` loads frame f's inputs and is called only
    for this rank's frames. With ``gather`` every rank but 0 ships each
    finished frame's mesh and visibility bits to rank 0 straight from device
    memory (NCCL point-to-point over NVLink; the small meta vector over
    gloo) and reads back only its rendered view. Rank 0 yields
    (frame_id, SceneBundle, image or None) for EVERY frame in order, images
    for its own frames; the other ranks yield (frame_id, None, image) for
    theirs. Without torch.distributed this is run_sequence over all frames."""
    import itertools

    import torch.distributed as dist

    from .sharding import bundle_from_export, frame_gather, frames_for_rank, merge_sharded

    if dist.is_available() and dist.is_initialized():
        rank, world = dist.get_rank(group), dist.get_world_size(group)
    else:
        rank, world = 0, 1
    mine = frames_for_rank(rank, world, n_frames)
    a, b = itertools.tee(map(source, mine))
    gatherer = frame_gather(group) if gather and world > 1 else None
    local = _run_local(cfg, rig, (p[0] for p in a), (p[1] for p in b), virtual, fallback_color,
                       iter(mine), lanes, export=gatherer is not None and rank != 0)

    def to_bundle(fid, meta, payload, ev):
        if ev is not None:
            ev.synchronize()
        return bundle_from_export(meta, payload, cfg, rig, fid)

    yield from merge_sharded(rank, world, n_frames, local, gatherer, to_bundle)


def sweep(cfg: PipelineConfig, rig, sils, axis: str, values) -> list:
    """run_frame per spacing value on fixed inputs (pipeline.py:223-243)."""
    if axis not in ("coarse_spacing", "fine_spacing"):
        raise ValueError(f"unknown sweep axis {axis!r}")
    if list(values) != sorted(values):
        raise ValueError("sweep values must be ascending")
    dsils = DeviceSilhouettes(rig, sils)
    rows = []
    for v in values:
        if axis == "coarse_spacing":
            run_cfg = replace(cfg, coarse_spacing=float(v), roi_margin=None, t_v=cfg.t_v)
            if run_cfg.fine_spacing > run_cfg.coarse_spacing:
                raise ValueError(f"coarse value {v} below fine_spacing")
        else:
            run_cfg = replace(cfg, fine_spacing=float(v), t_v=None)
        bundle = run_frame(run_cfg, rig, frames={c.id: None for c in rig}, sils=dsils)
        rows.append((float(v), bundle.timings))
    return rows


def sweep_csv(rows, path) -> None:
    import csv

    with open(path, "w", newline="", encoding="utf-8") as fh:
        w = csv.writer(fh)
        w.writerow(["value"] + [label for _, label in StageTimings.LABELS] + ["total"])
        for value, t in rows:
            w.writerow([value] + [f"{getattr(t, k):.3f}" for k, _ in StageTimings.LABELS]
                       + [f"{t.total:.3f}"])
