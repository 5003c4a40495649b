#!/usr/bin/env python
"""FVV frames/s benchmark (BASELINE.json metric) on the C3 volleyball workload.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

One step = one synthetic frame through B-1 sparse carve, B-2 CCL/filter/ROI,
B-3 ROI carve, C exact polygonisation, D-1 depth images, D-2 visibility and
one 1920x1080 virtual-view colour pass. Frames are sharded
across ranks (frame f -> rank f mod N, no collective on the data path:
weak scaling). Rank 0 prints one JSON line.

  value : frames/s, inputs resident in HBM, device time (CUDA events,
          barrier + synchronize on both sides, max over ranks), the K frames
          spread over --lanes executor lanes (thread + CUDA stream each);
          value_single_stream is the same K frames on one stream; stage_ms /
          roofline come from a further single-stream pass with the per-stage
          events read back
  e2e   : frames/s through the public API (pipeline.run_sequence =
          run_frame + render_view per frame) from pinned host buffers: H2D
          of every frame's silhouettes, the colour pass's zero-copy reads of
          the pinned colour frames, and D2H of the mesh, visibility flags
          and rendered image all inside the timed region
  --impl reference : the CPU oracle port of the reference pipeline
          (oracle/, C + OpenMP, all host threads), same workload and metric.
"""

from __future__ import annotations

import argparse
import gc
import json
import os
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

MEASURED_PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")
FALLBACK_HBM_GBS = 6650.0  # B200_PROFILING.md fallback, used only without MEASURED_PEAKS.json
METRIC = "FVV frames/sec (carve+CCL+mesh+color) at 1/2/4/8 B200; Gvoxel-projections/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=60,
                    help="timed frames (the reference arm: one full CPU frame per step)")
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="C3")
    ap.add_argument("--frames", type=int, default=4, help="distinct input frames per rank")
    ap.add_argument("--lanes", type=int, default=None,
                    help="concurrent executor lanes (threads + streams) per GPU; default 8, "
                         "3 for C4 (its 32 x 4K depth planes take 2.1 GB per executor)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--stage-json", default=None, help="write per-stage ms here (rank 0)")
    return ap.parse_args()


def self_launch(args):
    """``--gpus N`` without a torchrun environment: re-run this script as N
    frame-sharded ranks (one process per GPU) under torch.distributed.run and
    return its exit code; None when no launch is needed. Fails loudly when
    fewer than N GPUs are visible or a torchrun world disagrees with N."""
    if "WORLD_SIZE" in os.environ:
        ws = int(os.environ["WORLD_SIZE"])
        if ws != args.gpus:
            sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws}")
        return None
    if args.gpus <= 1 or args.impl == "reference":
        return None  # the reference arm runs on rank 0 only
    import socket

    import torch

    visible = torch.cuda.device_count()
    if visible < args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but only {visible} CUDA device(s) visible")
    s_ = socket.socket()
    s_.bind(("127.0.0.1", 0))
    port = s_.getsockname()[1]
    s_.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1", f"--master-port={port}",
           os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def dist_setup(args):
    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if torch.cuda.is_available():
        torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl" if torch.cuda.is_available() else "gloo")
    return rank, world, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def max_over_ranks(x, world):
    from paper_1903_11785_b200.sharding import reduce_max

    return reduce_max(x) if world > 1 else x


def sum_over_ranks(x, world):
    from paper_1903_11785_b200.sharding import reduce_sum

    return reduce_sum(x) if world > 1 else x


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.idx = gpu_index
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100", "-f", self.path],
                stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
        except Exception:  # noqa: BLE001
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:  # noqa: BLE001
            self.proc.kill()
        rows = []
        with open(self.path) as fh:
            for line in fh:
                parts = [p.strip() for p in line.split(",")]
                if len(parts) >= 9:
                    rows.append(parts)
        os.unlink(self.path)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = sorted(float(r[1]) for r in rows if r[1].replace(".", "").isdigit())
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in rows for n, v in zip(names, r[5:9]) if v.lower() == "active"})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None,
                "sm_max_mhz": float(rows[0][2]) if rows[0][2].replace(".", "").isdigit() else None,
                "reasons": reasons, "samples": len(rows)}


def peaks():
    try:
        with open(MEASURED_PEAKS) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json)", p
    except Exception:  # noqa: BLE001
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)", {}


# ---------------------------------------------------------------- inputs
def make_inputs(wl, frame_ids):
    """Silhouettes (N,H,W) uint8 and colour frames (N,H,W,3) uint8 on the GPU."""
    from paper_1903_11785_b200 import synthetic as S

    out = []
    for f in frame_ids:
        masks, frames = S.render_scene_device(wl.rig, wl.objects(f), shade=True)
        out.append((f, masks, frames))
    return out


# ---------------------------------------------------------------- b200 arm
def run_b200(args):
    import numpy as np
    import torch

    from paper_1903_11785_b200 import _lib, workloads

    rank, world, local = dist_setup(args)
    wl = workloads.get(args.workload)
    rig, cfg, virt = wl.rig, wl.cfg, wl.virtual
    cams = list(rig)
    ncam = len(cams)
    from paper_1903_11785_b200.sharding import frames_for_rank

    frame_ids = frames_for_rank(rank, world, world * args.frames)  # frame f -> rank f mod N
    inputs = make_inputs(wl, frame_ids)
    torch.cuda.synchronize()

    dev_frames = []
    for f, masks, frames in inputs:
        fb = frames.reshape(-1)
        foff = np.arange(ncam, dtype=np.int64) * (frames.shape[1] * frames.shape[2] * 3)
        dev_frames.append((masks, fb, foff))

    from paper_1903_11785_b200.executor import executor_for

    lanes = max(1, args.lanes)
    exs = [executor_for(cfg, rig, k) for k in range(lanes)]
    ex = exs[0]
    stage_names = ("sparse_carve", "noise_filter_roi", "dense_carve", "polygonize",
                   "depth_images", "visibility", "render")
    stage_sum = {k: 0.0 for k in stage_names}
    work = {"proj": 0, "tris": 0, "frames": 0, "nv": 0}

    nfr = len(dev_frames)

    def device_step(i, timed, lane_ex=None):
        # frame slot (i + i // lanes) mod F: lane k (steps k, k + lanes, ...)
        # walks through every input frame instead of re-running one
        masks, fb, foff = dev_frames[(i + i // lanes) % nfr]
        out = (lane_ex or ex).run(masks, virt, fb, foff)
        if timed:
            st = out.stats_raw
            for k, ms_ in zip(stage_names, st["ms"][:7]):
                stage_sum[k] += float(ms_)
            # algorithmic voxel-camera projections (hull.py:83-90): every voxel
            # of the stage grid and of every ROI grid against every camera
            work["proj"] += int(st["sparse_tests"] + st["dense_tests"]) * ncam
            work["tris"] += int(st["triangles"])
            work["nv"] = int(st["vertices"])
            work["frames"] += 1
            work["last"] = (int(st["sparse_tests"]), int(st["dense_tests"]))

    lib = _lib.load()
    # the timed passes do not read the per-stage event times back (~22 us of
    # host time per frame); a separate single-stream pass collects them
    for e in exs:
        e.stage_times = False
    # ---- single-stream pass (one CUDA stream, not the legacy default stream,
    # so frames replay as graphs) ----
    single = torch.cuda.Stream()
    with torch.cuda.stream(single):
        for i in range(args.warmup):
            device_step(i, False)
        torch.cuda.synchronize()
        barrier(world)
        s_start = torch.cuda.Event(enable_timing=True)
        s_end = torch.cuda.Event(enable_timing=True)
        s_start.record()
        for i in range(args.steps):
            device_step(i, False)
        s_end.record()
    torch.cuda.synchronize()
    barrier(world)
    ms_single = max_over_ranks(s_start.elapsed_time(s_end), world)
    # ---- per-stage device times (roofline inputs): the same K frames on the
    # same stream with the stage events read back ----
    ex.stage_times = True
    with torch.cuda.stream(single):
        for i in range(args.steps):
            device_step(i, True)
    torch.cuda.synchronize()
    ex.stage_times = False
    stage_ms = {k: v / args.steps for k, v in stage_sum.items()}

    # ---- timed region: K frames over `lanes` executors (one thread and one
    # CUDA stream each, frame i on lane i mod lanes), inputs resident in HBM ----
    import threading

    dev_index = torch.cuda.current_device()
    streams = [torch.cuda.Stream() for _ in range(lanes)]

    def run_lanes(n, base=0):
        errors = []

        def lane(k):
            try:
                torch.cuda.set_device(dev_index)
                with torch.cuda.stream(streams[k]):
                    for i in range(base + k, base + n, lanes):
                        device_step(i, False, exs[k])
            except BaseException as exc:  # noqa: BLE001
                errors.append(exc)

        cur = torch.cuda.current_stream()
        for st_ in streams:
            st_.wait_stream(cur)
        ths = [threading.Thread(target=lane, args=(k,)) for k in range(lanes)]
        for th in ths:
            th.start()
        for th in ths:
            th.join()
        for st_ in streams:
            cur.wait_stream(st_)
        if errors:
            raise errors[0]

    run_lanes(max(args.warmup, lanes) * lanes)  # every lane warm
    torch.cuda.synchronize()
    barrier(world)
    sampler = ClockSampler(local if "CUDA_VISIBLE_DEVICES" not in os.environ else
                           os.environ["CUDA_VISIBLE_DEVICES"].split(",")[local])
    sampler.start()
    launches0 = lib.fvv_launch_count()
    torch.cuda.synchronize()
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    gc.collect()
    gc.freeze()  # setup objects out of the collector's way
    gc.disable()  # as timeit: no collector pauses inside timed regions
    t_start.record()
    run_lanes(args.steps)
    t_end.record()
    torch.cuda.synchronize()
    gc.enable()
    launches = lib.fvv_launch_count() - launches0
    barrier(world)
    clocks = sampler.stop()
    ms_local = t_start.elapsed_time(t_end)
    ms = max_over_ranks(ms_local, world)

    total_frames = sum_over_ranks(args.steps, world)
    total_proj = sum_over_ranks(work["proj"], world)
    value = total_frames / (ms / 1e3)
    value_single = total_frames / (ms_single / 1e3)

    # ---- roofline of the dominant kernel: the
    # carve kernel (B-1 + B-3) has the largest GPU time per frame in the ncu
    # launch list (profiles/); north_star asks for it against the FFMA roofline
    hbm_peak, peak_src, _ = peaks()
    H, W = cams[0].image_height, cams[0].image_width
    roof_stages = stage_rooflines(stage_ms, work, ncam, H, W, hbm_peak, peak_src)
    roof = carve_roofline(stage_ms, work, ncam)
    for st_name in ("depth_images", "polygonize", "visibility", "render"):
        roof_stages[st_name] = roofline_for(st_name, stage_ms[st_name], work, ncam, H, W,
                                            hbm_peak, peak_src)
    attach_executed(roof_stages, stage_ms)

    # ---- e2e through the public API from pinned host memory ----
    e2e = None
    if not args.no_e2e:
        host = []
        for f, masks, frames in inputs:
            m_h = masks.cpu().pin_memory()
            f_h = frames.cpu().pin_memory()
            host.append((m_h, {c.id: f_h[k] for k, c in enumerate(cams)}))

        from paper_1903_11785_b200 import render as R
        from paper_1903_11785_b200 import sharding as SH
        from paper_1903_11785_b200.pipeline import run_sequence, run_sequence_sharded

        def consume(bundle, img):
            # what a viewer reads per frame: the merged mesh and the virtual view
            n = 0
            if bundle is not None:
                m = bundle.merged_mesh
                n += m.vertices.shape[0] + m.triangles.shape[0]
            if img is not None:
                n += img.color.shape[0]
            return n

        def sequence(nsteps):
            """This rank's share of an nsteps x world frame sequence: frame f
            on rank f mod N; at N > 1 every frame's mesh + visibility is
            gathered to rank 0 over NCCL (run_sequence_sharded)."""
            if world == 1:
                # input (i + i // 2 lanes) mod F: each lane runs its frames on two
                # executors in turn, and this way both of them meet every input
                # within 2 F rounds (the warm-up covers that: no executor sees a
                # new input, i.e. no capacity growth or graph capture, in the
                # timed run whatever lane the sequence runner starts it on)
                idx = [(i + i // (2 * lanes)) % len(host) for i in range(nsteps)]
                fr = [host[k][1] for k in idx]
                ms_ = [host[k][0] for k in idx]
                for bundle, img in run_sequence(cfg, rig, fr, ms_, virt, lanes=lanes):
                    yield bundle, img
                return

            def source(f):  # the j-th frame of this rank is global frame rank + j * N
                j = f // world
                m_h, fr_h = host[(j + j // (2 * lanes)) % len(host)]
                return fr_h, m_h

            for _, bundle, img in run_sequence_sharded(cfg, rig, source, nsteps * world, virt,
                                                       lanes=lanes):
                yield bundle, img

        trace = os.environ.get("FVV_BENCH_TRACE")

        def run_e2e(nsteps):
            total = 0
            t_prev = time.perf_counter()
            gaps = []
            c_prev, m_prev = time.process_time(), time.thread_time()
            d2h0 = R.D2H_BYTES["results"]
            for bundle, img in sequence(nsteps):
                consume(bundle, img)
                t_now = time.perf_counter()
                gaps.append(round((t_now - t_prev) * 1e3, 2))
                t_prev = t_now
            if trace:
                hs = torch.cuda.host_memory_stats()
                print(f"e2e intervals (ms): {gaps}", file=sys.stderr)
                print(f"host CPU ms per frame (all threads): "
                      f"{(time.process_time() - c_prev) * 1e3 / nsteps:.3f}; caller thread: "
                      f"{(time.thread_time() - m_prev) * 1e3 / nsteps:.3f}", file=sys.stderr)
                print("host allocator: " + ", ".join(
                    f"{k}={hs[k]}" for k in sorted(hs) if k.startswith(("num_host", "allocations.",
                                                                       "active_requests"))),
                      file=sys.stderr)
            total = R.D2H_BYTES["results"] - d2h0  # bytes read back (pinned blocks)
            return total

        # warm-up covers every distinct input on every lane (buffer growth,
        # pinned readback pool) so the timed steps are steady state
        # (>= 6 frames per executor, two executors per lane: host-planned,
        # device-planned, graph capture, and capacity growth over the cycled
        # frames all happen before the timed region)
        run_e2e(max(args.warmup, 4 * len(host) + 2, 24 * lanes + 2))
        torch.cuda.synchronize()
        barrier(world)
        R.H2D_BYTES["frames"] = R.H2D_BYTES["masks"] = 0
        g0 = SH.GATHER_BYTES["payload"]
        gc.collect()
        gc.disable()
        t0 = time.perf_counter()
        d2h = run_e2e(args.steps)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        gc.enable()
        barrier(world)
        h2d = int((R.H2D_BYTES["masks"] + R.H2D_BYTES["frames"]) / args.steps)
        e2e_ms = max_over_ranks((t1 - t0) * 1e3, world)
        gathered = SH.GATHER_BYTES["payload"] - g0
        e2e = {"value": round(total_frames / (e2e_ms / 1e3), 3), "unit": "frames/s",
               "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": int((d2h + gathered) / args.steps),
               "ms_per_step": round(e2e_ms / args.steps, 3),
               "api": f"pipeline.run_sequence (run_frame + render_view per frame) on the "
                      f"native sequence runner (csrc/seq.cu: {lanes} C++ lanes, each with its "
                      "own streams and two frame executors); silhouettes uploaded per frame by "
                      "its lane, pinned colour frames sampled in place (zero-copy: h2d counts the 12 B of "
                      "bilinear taps per sourced pixel), results read back on a readback "
                      "stream as one pinned block per frame (virtual view as colour + an "
                      "int8 source/coverage code), pinned host inputs" +
                      ("" if world == 1 else
                       f"; frame-sharded over {world} ranks (run_sequence_sharded): every "
                       "frame's mesh + visibility sent to rank 0 over NCCL and read back "
                       "there (rank 0's d2h includes them), images read back per rank")}
        if world > 1:
            e2e["gather_bytes_rank0"] = int(gathered)

    # ---- CPU baseline: the oracle port on this box's host cores, rank 0, N=1 ----
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(wl, inputs[0])

    if rank == 0:
        line = {
            "metric": METRIC,
            "value": round(value, 3),
            "unit": "frames/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": round(ms / args.steps, 4),
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "f64",
            "data": "synthetic (GPU ray-cast ellipsoid figures, BASELINE C3)",
            "config": {"workload": f"{wl.name}: {wl.description}", "cameras": ncam,
                       "image": f"{W}x{H}", "coarse_mm": cfg.coarse_spacing,
                       "fine_mm": cfg.fine_spacing, "virtual_view": "1920x1080",
                       "frames_cycled": args.frames,
                       "l2": f"inputs cycle over {args.frames} frames x "
                             f"{(ncam * H * W * 4) / 1e6:.0f} MB (> 126 MB L2)",
                       "parallelism": f"frame-sharded x{world}, {lanes} executor lanes "
                                      f"per GPU",
                       "timing": "value: K frames over the lanes (CUDA events, barrier + sync "
                                 "both sides); value_single_stream: the same K frames on one "
                                 "stream; stage_ms / roofline: a further single-stream pass of "
                                 "them with the per-stage events read back (the timed passes "
                                 "skip that readout); Python's collector paused inside timed "
                                 "regions (as timeit)"},
            "value_single_stream": round(value_single, 3),
            "lanes": lanes,
            "gvoxel_proj_per_s": round(total_proj / (ms / 1e3) / 1e9, 2),
            "triangles_per_frame": int(work["tris"] / max(args.steps, 1)),
            "stage_ms": {k: round(v, 4) for k, v in stage_ms.items()},
            "roofline": roof,
            "roofline_stages": roof_stages,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": int(launches),
            "clocks": clocks,
        }
        print(json.dumps(line))
        if args.stage_json:
            with open(args.stage_json, "w") as fh:
                json.dump(line, fh, indent=2)


def roofline_for(stage, ms, work, ncam, H, W, hbm_peak, peak_src):
    """Algorithmic bytes of the dominant stage's kernels per launch / time."""
    nvox_c, nvox_f = work["last"]
    tris = work["tris"] // max(work["frames"], 1)
    verts = work["nv"]
    sil_bytes = ncam * H * ((W + 31) // 32) * 4
    per_stage = {
        # silhouette planes read once + occupancy bits written
        "sparse_carve": ("fvv_carve (B-1)", sil_bytes + nvox_c / 8),
        "dense_carve": ("fvv_carve (B-3)", sil_bytes + nvox_f / 8),
        # occupancy bits + int32 label per voxel
        "noise_filter_roi": ("fvv_ccl26", nvox_c / 8 + 4 * nvox_c),
        # occupancy bits read, vertices + triangles written, silhouettes read
        "polygonize": ("fvv_mesh_prepare+emit", nvox_f / 8 + 24 * verts + 12 * tris + sil_bytes),
        # every camera's float64 depth plane written once, mesh read once per camera
        "depth_images": ("fvv_rasterize (16 cams)", ncam * H * W * 8 + ncam * (24 * verts +
                                                                             12 * tris)),
        # centroid depth lookups + visibility bits
        "visibility": ("fvv_classify", ncam * tris * 8 + ncam * tris / 8 + 24 * verts +
                       12 * tris),
        # virtual view depth + id planes, colour/source written, 4 texel reads per pixel
        "render": ("fvv_rasterize+fvv_render_view (virtual)", 1920 * 1080 * (8 + 4 + 3 + 4 + 1)),
    }
    kernel, nbytes = per_stage.get(stage, (stage, 0.0))
    achieved = nbytes / (ms / 1e3) / 1e9
    traffic = None  # measured DRAM bytes: attach_executed (profiles/exec_counters.json)
    return {"bound": "hbm", "kernel": kernel, "stage": stage, "achieved": round(achieved, 2),
            "peak": hbm_peak, "peak_source": peak_src, "unit": "GB/s",
            "frac": round(achieved / hbm_peak, 5), "traffic": traffic,
            "traffic_source": None,
            "algorithmic_bytes": int(nbytes), "ms_per_launch": round(ms, 4)}


def fp32_peak_tflops():
    """148 SMs x 128 FP32 lanes x 2 FLOP x the max SM clock (MEASURED_PEAKS.json
    has no FP32 figure; the clock is the driver-measured sm_max_mhz)."""
    import torch

    props = torch.cuda.get_device_properties(0)
    sm_mhz = 1965.0
    try:
        with open(MEASURED_PEAKS) as fh:
            sm_mhz = float(json.load(fh).get("sm_max_mhz", sm_mhz))
    except Exception:  # noqa: BLE001
        pass
    basis = (f"derived: {props.multi_processor_count} SMs x 128 FP32 lanes x 2 FLOP x "
             f"{sm_mhz:.0f} MHz (sm_max_mhz, MEASURED_PEAKS.json; it holds no FP32 figure)")
    return props.multi_processor_count * FP32_LANES_PER_SM * 2 * sm_mhz * 1e6 / 1e12, basis


def carve_roofline(stage_ms, work, ncam):
    """The carve kernel (B-1 stage grid + B-3 ROI grids, one launch each per
    frame) against the FP32 FFMA roofline: algorithmic FLOP = every voxel x
    every camera x 26 FLOP (BASELINE.md 2 / SURVEY.md 8d: 13 FMA-pipe ops per
    voxel-projection), as hull.py:83-90 evaluates them; tile culling and the
    early exit execute fewer, so the fraction is of the algorithmic work."""
    nvox_c, nvox_f = work["last"]
    proj = (nvox_c + nvox_f) * ncam
    ms = stage_ms["sparse_carve"] + stage_ms["dense_carve"]
    peak, basis = fp32_peak_tflops()
    achieved = FLOP_PER_PROJECTION * proj / (ms / 1e3) / 1e12
    traffic = None  # DRAM bytes per launch (B-1 + B-3 stages of profiles/exec_counters.json)
    try:
        with open(EXEC_COUNTERS) as fh:
            st_ = json.load(fh)["stages"]
        traffic = int((st_["B-1"]["dram_mb"] + st_["B-3"]["dram_mb"]) * 1e6 / 2)
    except Exception:  # noqa: BLE001
        pass
    return {"bound": "fp32", "kernel": "carve_kernel (B-1 stage grid + B-3 ROI grids)",
            "stage": "sparse_carve + dense_carve", "achieved": round(achieved, 3),
            "peak": round(peak, 2), "unit": "TFLOP/s", "frac": round(achieved / peak, 4),
            "traffic": traffic,
            "traffic_source": "profiles/exec_counters.json (ncu --set full: dram bytes of the B-1 and B-3 stages, prep + classification + octants + float64 queue, per launch)",
            "peak_source": basis, "launches_per_frame": 2,
            "algorithmic_flop_per_launch": int(FLOP_PER_PROJECTION * proj / 2),
            "voxel_projections_per_frame": int(proj), "ms_per_launch": round(ms / 2, 4),
            "note": "tensor cores unused: no stage is a dense contraction (north_star)"}


FP32_LANES_PER_SM = 128  # B200: 128 FP32 lanes per SM
FLOP_PER_PROJECTION = 26  # 13 FMA-pipe ops per voxel-projection


def stage_rooflines(stage_ms, work, ncam, H, W, hbm_peak, peak_src):
    """BASELINE.md 2's per-stage rooflines: the carves against FP32 issue in
    voxel-projections/s (algorithmic projections = every voxel x every
    camera, as hull.py:83-90 computes them; culling and early exits do not
    reduce the count), CCL against HBM."""
    import torch

    props = torch.cuda.get_device_properties(0)
    sm_mhz = 1965.0
    try:
        with open(MEASURED_PEAKS) as fh:
            sm_mhz = float(json.load(fh).get("sm_max_mhz", sm_mhz))
    except Exception:  # noqa: BLE001
        pass
    fp32_tflops = props.multi_processor_count * FP32_LANES_PER_SM * 2 * sm_mhz * 1e6 / 1e12
    proj_peak = fp32_tflops * 1e12 / FLOP_PER_PROJECTION  # voxel-projections/s
    nvox_c, nvox_f = work["last"]
    out = {}
    for stage, nvox in (("sparse_carve", nvox_c), ("dense_carve", nvox_f)):
        ms = stage_ms[stage]
        rate = nvox * ncam / (ms / 1e3)
        out[stage] = {"bound": "fp32_issue", "achieved": round(rate / 1e12, 4),
                      "peak": round(proj_peak / 1e12, 4), "unit": "T voxel-proj/s",
                      "frac": round(rate / proj_peak, 4), "ms": round(ms, 4),
                      "peak_basis": f"{props.multi_processor_count} SMs x 128 FP32 x 2 x "
                                    f"{sm_mhz:.0f} MHz / 26 FLOP"}
    ms = stage_ms["noise_filter_roi"]
    ccl_bytes = nvox_c / 8 + 4 * nvox_c
    gbs = ccl_bytes / (ms / 1e3) / 1e9
    out["noise_filter_roi"] = {"bound": "hbm", "achieved": round(gbs, 2), "peak": hbm_peak,
                               "unit": "GB/s", "frac": round(gbs / hbm_peak, 5),
                               "ms": round(ms, 4), "algorithmic_bytes": int(ccl_bytes),
                               "peak_source": peak_src}
    return out


EXEC_COUNTERS = os.path.join(ROOT, "profiles", "exec_counters.json")
STAGE_OF = {"sparse_carve": "B-1", "noise_filter_roi": "B-2", "dense_carve": "B-3",
            "polygonize": "C", "depth_images": "D-1", "visibility": "D-2", "render": "E"}


def attach_executed(roof_stages, stage_ms):
    """Executed-work counters per stage from the committed ncu capture of one
    C3 frame (profiles/exec_counters.json, scripts/exec_counters.py): FP32 /
    FP64 pipe and issue utilisation, executed FLOP rates, DRAM bytes per
    frame (the stage's measured traffic) and L2 / L1-gather throughput. C is
    bounded by the FP64 pipe (the float64 isovalue chain) and B-2 by launch /
    dependency latency (a few thousand ON voxels), so those two rooflines are
    stated against them."""
    try:
        with open(EXEC_COUNTERS) as fh:
            ex = json.load(fh)
    except Exception:  # noqa: BLE001
        return
    peaks_ = ex.get("peaks", {})
    for stage, key in STAGE_OF.items():
        c = ex.get("stages", {}).get(key)
        if not c or stage not in roof_stages:
            continue
        keep = ("us", "launches", "fp32_tflops", "fp64_tflops", "fma_pipe_pct", "fp64_pipe_pct",
                "issue_pct", "dram_mb", "dram_gbps", "l2_gbps", "l1_gather_gbps")
        r = roof_stages[stage]
        r["executed"] = {k: c[k] for k in keep if k in c}
        r["executed"]["source"] = "profiles/exec_counters.json (ncu --set full, cold caches, serialised)"
        r["traffic"] = int(c["dram_mb"] * 1e6) if "dram_mb" in c else r.get("traffic")
        r["traffic_source"] = "profiles/exec_counters.json (dram__bytes read+write, per frame)"
    if "polygonize" in roof_stages and "C" in ex.get("stages", {}):
        c = ex["stages"]["C"]
        pk = peaks_.get("fp64_tflops", 37.22)
        roof_stages["polygonize"].update({
            "bound": "fp64", "unit": "TFLOP/s", "achieved": c.get("fp64_tflops"), "peak": pk,
            "frac": round(c.get("fp64_tflops", 0.0) / pk, 4),
            "peak_source": "148 SMs x 64 DFMA lanes x 2 x 1965 MHz",
            "note": "executed FP64 FLOP rate of the C kernels (ncu); the float64 isovalue "
                    "chain of mesh.py:231-272 dominates"})
    if "noise_filter_roi" in roof_stages:
        r = roof_stages["noise_filter_roi"]
        r.update({"bound": "latency", "ms": round(stage_ms["noise_filter_roi"], 4),
                  "note": "dependency-latency bound: a few thousand ON voxels through a "
                          "rank scan, a run-based union-find, a root scan and stats in one "
                          "cooperative launch with grid barriers (ccl_fused_kernel), then "
                          "the ROI planner; its HBM fraction (algorithmic bytes / time) is "
                          "kept in 'frac'"})


# ---------------------------------------------------------------- CPU arm
def cpu_frame(wl, masks_np, frames_np):
    """One frame through the CPU oracle (B-1..D-2 + virtual colour pass)."""
    import oracle as O

    cfg = wl.cfg
    cams = list(wl.rig)
    out = O.run_frame(cams, masks_np, cfg.stage_lo, cfg.stage_hi, cfg.coarse_spacing,
                      cfg.fine_spacing, cfg.min_views, cfg.t_small, cfg.t_large, cfg.roi_margin,
                      cfg.t_v)
    v, t, _ = out["merged"]
    if len(t):
        O.render_view(v, t, cams, frames_np, out["visibility"], wl.virtual)
    return out


def cpu_baseline(wl, inp):
    _, masks, frames = inp
    masks_np = [m.cpu().numpy().astype(bool) for m in masks]
    fr = frames.cpu().numpy()
    frames_np = {c.id: fr[k] for k, c in enumerate(wl.rig)}
    t0 = time.perf_counter()
    cpu_frame(wl, masks_np, frames_np)
    dt = time.perf_counter() - t0
    return {"value": round(1.0 / dt, 5), "unit": "frames/s", "cores": os.cpu_count(),
            "kind": "port",
            "sample": f"1 {wl.name} frame (B-1..D-2 + 1080p colour pass) through oracle/ "
                      f"(C restatement of the reference, OpenMP {os.cpu_count()} threads), "
                      f"{dt:.2f} s"}


def _maps_product_library():
    try:
        with open("/proc/self/maps") as fh:
            return "libfvv.so" in fh.read()
    except OSError:
        return None


def run_reference(args):
    """The reference arm: the CPU oracle port of the reference pipeline
    (oracle/, C + OpenMP on every host thread) over the same workload, metric
    and frames as the GPU arm. Its inputs come from the HOST scene generator
    (synthetic.render_scene: numpy ray casts), so nothing of the product
    (libfvv.so, CUDA) is loaded on this path; the line records that."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    if rank != 0:
        return
    from concurrent.futures import ThreadPoolExecutor

    from paper_1903_11785_b200 import synthetic as S
    from paper_1903_11785_b200 import workloads

    wl = workloads.get(args.workload)
    ids = list(range(max(1, args.frames)))  # the frames the GPU arm cycles (rank 0, N = 1)
    t0 = time.perf_counter()
    with ThreadPoolExecutor(max_workers=min(len(ids), os.cpu_count() or 1)) as pool:
        inputs = list(pool.map(lambda f: S.render_scene(wl.rig, wl.objects(f)), ids))
    t_gen = time.perf_counter() - t0
    for i in range(args.warmup):
        cpu_frame(wl, *inputs[i % len(inputs)])
    t0 = time.perf_counter()
    for i in range(args.steps):
        cpu_frame(wl, *inputs[i % len(inputs)])
    dt = time.perf_counter() - t0
    value = args.steps / dt
    print(json.dumps({
        "metric": METRIC, "value": round(value, 5), "unit": "frames/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(dt / args.steps * 1e3, 2),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (host ray-cast ellipsoid figures, BASELINE C3)", "impl": "reference",
        "config": {"workload": f"{wl.name}: {wl.description}", "cameras": len(wl.rig),
                   "frames_cycled": len(ids), "frame_ids": ids, "virtual_view": "1920x1080"},
        "cpu_baseline": {"value": round(value, 5), "unit": "frames/s", "cores": os.cpu_count(),
                         "kind": "port",
                         "sample": f"every step = 1 full frame (B-1..D-2 + 1080p colour pass) "
                                   f"through oracle/ (C restatement of the reference pipeline, "
                                   f"OpenMP {os.cpu_count()} threads), frames {ids} cycled"},
        "e2e": {"value": round(value, 5), "unit": "frames/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "inputs": f"synthetic.render_scene on the host ({t_gen:.1f} s, outside the timed region)",
        "product_library_loaded": _maps_product_library(),
    }))


def main():
    args = parse()
    if args.lanes is None:
        args.lanes = 3 if args.workload == "C4" else 8
    rc = self_launch(args)
    if rc is not None:
        sys.exit(rc)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
