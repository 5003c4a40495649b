"""Pinned host<->device copy bandwidth on this box (H2D, D2H, both at once)."""
import torch

n = 34 << 20
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d = torch.empty(n, dtype=torch.uint8, device="cuda")
d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for name, ops in (("h2d", [(s1, d, h)]), ("d2h", [(s2, h2, d2)]),
                  ("both", [(s1, d, h), (s2, h2, d2)])):
    for rep in range(2):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for st, dst, src in ops:
            st.wait_event(e0)
            with torch.cuda.stream(st):
                for _ in range(10):
                    dst.copy_(src, non_blocking=True)
        for st, _, _ in ops:
            torch.cuda.current_stream().wait_stream(st)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
    print(f"{name}: {10 * n * len(ops) / ms / 1e6:.1f} GB/s total ({ms / 10:.3f} ms per 34 MB)")
