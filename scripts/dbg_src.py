import sys; sys.path.insert(0, '/root/repo')
import numpy as np, torch, ctypes
from paper_1903_11785_b200 import render as R, _lib
class C:
    def __init__(s, i): s.id = i
for nrank, n in [(3, 3)]:
    rig = [C(i) for i in range(nrank)]
    vis = {i: np.random.default_rng(i).random(n) < 0.3 for i in range(nrank)}
    bits, stride = R._vis_bits_from_dict(vis, rig, n, torch.device("cuda"))
    try:
        src = R.sources_device(list(range(nrank)), rig, bits, stride, n)
        torch.cuda.synchronize()
        print(nrank, n, "ok", src[:5].tolist())
    except Exception as e:
        print(nrank, n, "FAIL", e); break
