"""Single-stream executor frames/s with the host-planned path, device-planned
frames without graphs, and device-planned frames replayed as CUDA graphs.

    python scripts/plan_modes.py   (runs itself once per FVV_* setting)
"""
import os
import subprocess
import sys
import time

if len(sys.argv) > 1:
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import numpy as np
    import torch

    from paper_1903_11785_b200 import synthetic as S, workloads
    from paper_1903_11785_b200.executor import executor_for

    wl = workloads.get("C3")
    ins = []
    for fr in range(4):
        m, fs = S.render_scene_device(wl.rig, wl.objects(fr))
        ins.append((m, fs.reshape(-1)))
    foff = np.arange(len(wl.rig), dtype=np.int64) * (1920 * 1080 * 3)
    ex = executor_for(wl.cfg, wl.rig)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for i in range(8):
            ex.run(ins[i % 4][0], wl.virtual, ins[i % 4][1], foff)
        torch.cuda.synchronize()
        n = 200
        t0 = time.perf_counter()
        for i in range(n):
            out = ex.run(ins[i % 4][0], wl.virtual, ins[i % 4][1], foff)
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / n
    print(f"{sys.argv[1]:>12}: {1 / dt:7.1f} frames/s ({dt * 1e3:.3f} ms/frame) "
          f"stats {out.stats()['triangles']} tris, ms {[round(float(x), 3) for x in out.stats_raw['ms']]}")
else:
    for name, env in (("host-planned", {"FVV_DEVICE_PLAN": "0"}),
                      ("device", {"FVV_FRAME_GRAPH": "0"}), ("device+graph", {})):
        subprocess.run([sys.executable, __file__, name], env={**os.environ, **env,
                                                                "FVV_PLAN_DEBUG": "1"})
