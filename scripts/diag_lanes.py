"""Device-resident throughput with 1 vs 2 executor lanes (threads + streams)."""
import sys, os, time, threading
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1903_11785_b200 import workloads, synthetic as S
from paper_1903_11785_b200.executor import executor_for
wl = workloads.get("C3"); cams = list(wl.rig)
inputs = [S.render_scene_device(wl.rig, wl.objects(f), shade=True) for f in range(4)]
foff = np.arange(16, dtype=np.int64) * (1080 * 1920 * 3)
def lane_run(k, frames, stream, ex):
    torch.cuda.set_device(0)
    with torch.cuda.stream(stream):
        for i in frames:
            m, fr = inputs[i % 4]
            ex.run(m, wl.virtual, fr.reshape(-1), foff)
for lanes in (1, 2, 3):
    exs = [executor_for(wl.cfg, wl.rig, k) for k in range(lanes)]
    streams = [torch.cuda.Stream() for _ in range(lanes)]
    for rep in range(3):
        n = 60
        torch.cuda.synchronize(); t0 = time.perf_counter()
        ths = [threading.Thread(target=lane_run, args=(k, range(k, n, lanes), streams[k], exs[k])) for k in range(lanes)]
        for t in ths: t.start()
        for t in ths: t.join()
        torch.cuda.synchronize(); t1 = time.perf_counter()
        print(f"lanes {lanes}: {n / (t1 - t0):.1f} frames/s")
