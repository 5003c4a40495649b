"""Executed-work counters per kernel and per pipeline stage from an
`ncu --set full` capture of one frame (scripts/gpu/ncu_frame.sh, which runs
scripts/profile_frame.py under --profile-from-start off):

    python scripts/exec_counters.py gpurun_out/r2_frame_full.ncu-rep profiles/r2_exec_counters.json

Per kernel: device time (ncu replay: cold caches, serialised), executed FP32
and FP64 floating-point work (FFMA counted as 2 FLOP, FADD/FMUL as 1) and the
rates they reach, FMA / FP64 pipe utilisation, issue-slot utilisation, DRAM
bytes, L2 sectors and L1 global-load sectors (the gathers) with their
throughputs. Stages follow the executor's launch order (csrc/frame.cu):
B-1 sparse carve, B-2 CCL/ROI, B-3 dense carve, C polygonize, D-1 depth
images (16 cameras), D-2 visibility, E virtual view (raster + colour). Run
the captured program with FVV_FORK=0 (scripts/gpu/ncu_frame.sh does) so the
launches come in that order.
"""
import csv
import io
import json
import subprocess
import sys

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1.0,
         "ms": 1e3, "s": 1e6}
FP32_PEAK = 148 * 128 * 2 * 1.965e9 / 1e12  # TFLOP/s (FFMA lanes x 2 x sm_max_mhz)
FP64_PEAK = 148 * 64 * 2 * 1.965e9 / 1e12   # ncu: 64 DFMA/cycle/SM peak_sustained
HBM_PEAK = 6533.5                            # GB/s, MEASURED_PEAKS.json


def load(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def stage_of(names):
    """Stage label per launch, from the executor's launch order."""
    out, stage, carves, rasters = [], "B-1", 0, 0
    for n in names:
        if n.startswith("pack"):
            stage = "B-1"
        elif n.startswith("carve_prep"):
            carves += 1
            stage = "B-1" if carves == 1 else "B-3"
        elif "WordRank" in n or n.startswith("ccl_fused"):
            stage = "B-2"
        elif n.startswith("mesh_transpose"):
            stage = "C"
        elif n.startswith("raster_prep") or n.startswith("raster_vertex"):
            # the executor enqueues the virtual view's raster (E) right after
            # C (a side-stream branch; FVV_FORK=0 keeps it in the chain), then
            # D-1's; the colour pass follows D-2
            rasters += 1
            stage = "E" if rasters == 1 else "D-1"
        elif n.startswith("classify"):
            stage = "D-2"
        elif n.startswith("render_count") or n.startswith("render_color"):
            stage = "E"
        out.append(stage)
    return out


def main():
    rep, dst = sys.argv[1], sys.argv[2]
    h, units, rows = load(rep)
    col = {k: i for i, k in enumerate(h)}

    def val(r, k, scale=True):
        v = r[col[k]].replace(",", "")
        try:
            x = float(v)
        except ValueError:
            return 0.0
        return x * SCALE.get(units[col[k]], 1.0) if scale else x

    names = [r[col["Kernel Name"]].replace("void ", "").split("(")[0] for r in rows]
    stages = stage_of(names)
    kernels = []
    for r, name, st in zip(rows, names, stages):
        us = val(r, "gpu__time_duration.sum")
        cyc = val(r, "smsp__cycles_elapsed.avg", False)

        def ops(op):
            return val(r, f"smsp__sass_thread_inst_executed_op_{op}_pred_on.sum.per_cycle_elapsed",
                       False) * cyc

        f32 = 2 * ops("ffma") + ops("fadd") + ops("fmul")
        f64 = 2 * ops("dfma") + ops("dadd") + ops("dmul")
        dram = val(r, "dram__bytes_read.sum") + val(r, "dram__bytes_write.sum")
        l2 = 32 * val(r, "lts__t_sectors.sum", False)
        l1 = 32 * val(r, "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", False)
        s = us * 1e-6
        kernels.append({
            "kernel": name, "stage": st, "us": round(us, 2),
            "fp32_gflop": round(f32 / 1e9, 4), "fp32_tflops": round(f32 / s / 1e12, 3),
            "fp64_gflop": round(f64 / 1e9, 4), "fp64_tflops": round(f64 / s / 1e12, 3),
            "fma_pipe_pct": round(val(r, "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", False), 1),
            "fp64_pipe_pct": round(val(r, "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", False), 1),
            "issue_pct": round(val(r, "smsp__issue_active.avg.pct_of_peak_sustained_active", False), 1),
            "warps_active_pct": round(val(r, "sm__warps_active.avg.pct_of_peak_sustained_active", False), 1),
            "dram_mb": round(dram / 1e6, 3), "dram_gbps": round(dram / s / 1e9, 1),
            "l2_mb": round(l2 / 1e6, 3), "l2_gbps": round(l2 / s / 1e9, 1),
            "l2_hit_pct": round(val(r, "lts__t_sector_hit_rate.pct", False), 1),
            "l2_throughput_pct": round(val(r, "lts__throughput.avg.pct_of_peak_sustained_elapsed", False), 1),
            "l1_gather_mb": round(l1 / 1e6, 3), "l1_gather_gbps": round(l1 / s / 1e9, 1),
            "l1_hit_pct": round(val(r, "l1tex__t_sector_pipe_lsu_mem_global_op_ld_hit_rate.pct", False), 1),
            "smem_wavefronts": int(val(r, "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", False)),
        })
    agg = {}
    for k in kernels:
        a = agg.setdefault(k["stage"], {"us": 0.0, "fp32_gflop": 0.0, "fp64_gflop": 0.0,
                                        "dram_mb": 0.0, "l2_mb": 0.0, "l1_gather_mb": 0.0,
                                        "_fma": 0.0, "_fp64": 0.0, "_issue": 0.0, "launches": 0})
        a["us"] += k["us"]
        a["launches"] += 1
        for f in ("fp32_gflop", "fp64_gflop", "dram_mb", "l2_mb", "l1_gather_mb"):
            a[f] += k[f]
        a["_fma"] += k["fma_pipe_pct"] * k["us"]
        a["_fp64"] += k["fp64_pipe_pct"] * k["us"]
        a["_issue"] += k["issue_pct"] * k["us"]
    stages_out = {}
    for st, a in agg.items():
        s = a["us"] * 1e-6
        stages_out[st] = {
            "us": round(a["us"], 1), "launches": a["launches"],
            "fp32_tflops": round(a["fp32_gflop"] * 1e9 / s / 1e12, 3),
            "fp32_frac_of_peak": round(a["fp32_gflop"] * 1e9 / s / 1e12 / FP32_PEAK, 4),
            "fp64_tflops": round(a["fp64_gflop"] * 1e9 / s / 1e12, 3),
            "fp64_frac_of_peak": round(a["fp64_gflop"] * 1e9 / s / 1e12 / FP64_PEAK, 4),
            "fma_pipe_pct": round(a["_fma"] / a["us"], 1),
            "fp64_pipe_pct": round(a["_fp64"] / a["us"], 1),
            "issue_pct": round(a["_issue"] / a["us"], 1),
            "dram_mb": round(a["dram_mb"], 2), "dram_gbps": round(a["dram_mb"] * 1e6 / s / 1e9, 1),
            "dram_frac_of_peak": round(a["dram_mb"] * 1e6 / s / 1e9 / HBM_PEAK, 4),
            "l2_gbps": round(a["l2_mb"] * 1e6 / s / 1e9, 1),
            "l1_gather_gbps": round(a["l1_gather_mb"] * 1e6 / s / 1e9, 1),
        }
    doc = {"source": rep, "frame": "C3 frame 1 after 3 warm-up frames (scripts/profile_frame.py)",
           "note": "ncu --set full replays each launch with cold caches, serialised: absolute "
                   "times exceed the warm, overlapped bench numbers; shares and rates compare",
           "peaks": {"fp32_tflops": round(FP32_PEAK, 2), "fp64_tflops": round(FP64_PEAK, 2),
                     "hbm_gbps": HBM_PEAK,
                     "basis": "148 SMs x (128 FFMA | 64 DFMA lanes) x 2 x 1965 MHz; HBM measured"},
           "stages": stages_out, "kernels": kernels}
    with open(dst, "w") as fh:
        json.dump(doc, fh, indent=1)
    for st, a in stages_out.items():
        print(st, a)


if __name__ == "__main__":
    main()
