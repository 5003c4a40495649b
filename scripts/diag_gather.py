import sys, os, time, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1903_11785_b200 import _lib, pipeline as P
rt = ctypes.CDLL("libcudart.so.12") if False else None
n = 16; sz = 1920 * 1080 * 3
big = torch.empty(n * sz, dtype=torch.uint8).pin_memory()
views = [big[i * sz:(i + 1) * sz] for i in range(n)]
d = torch.empty(n * sz, dtype=torch.uint8, device="cuda")
s = torch.cuda.Stream()
keep = []
for trial in range(4):
    torch.cuda.synchronize(); t = time.perf_counter()
    P._gather_to_device([(v.data_ptr(), v.numel()) for v in views], d, s, keep)
    t1 = time.perf_counter(); torch.cuda.synchronize(); t2 = time.perf_counter()
    print(f"gather: enqueue {1e3*(t1-t):.3f} ms, total {1e3*(t2-t):.3f} ms")
for trial in range(2):
    torch.cuda.synchronize(); t = time.perf_counter()
    with torch.cuda.stream(s):
        for i, v in enumerate(views):
            d[i * sz:(i + 1) * sz].copy_(v, non_blocking=True)
    t1 = time.perf_counter(); torch.cuda.synchronize(); t2 = time.perf_counter()
    print(f"torch: enqueue {1e3*(t1-t):.3f} ms, total {1e3*(t2-t):.3f} ms")
print("is_pinned", big.is_pinned(), views[3].is_pinned())
