"""Deferred-voxel counts and timing of fvv_carve on a C3 frame (coarse
stage grid and the frame's ROI grids)."""
import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1903_11785_b200 import workloads, synthetic as S, _lib
from paper_1903_11785_b200._device import DeviceSilhouettes, stream_handle, grid_table
from paper_1903_11785_b200.executor import FrameExecutor
from paper_1903_11785_b200.hull import words_for
wl = workloads.get("C3")
masks, frames = S.render_scene_device(wl.rig, wl.objects(0))
ex = FrameExecutor(wl.cfg, wl.rig)
out = ex.run(masks)
ds = DeviceSilhouettes(wl.rig, masks)
lib = _lib.load()
wsb = int(lib.fvv_carve_workspace_bytes(_lib.host_ptr(ds.cams), ctypes.c_int(ds.ncam)))
ws = torch.zeros(wsb, dtype=torch.uint8, device="cuda")
coarse = grid_table([wl.cfg.coarse_spec()])
for name, tab in (("coarse", coarse), ("fine", np.ascontiguousarray(out.grids))):
    nvox = [int(np.prod(g["dims"])) for g in tab]
    words = [words_for(n) for n in nvox]
    off = np.zeros(len(tab), dtype=np.int64); off[1:] = np.cumsum(words)[:-1]
    bits = torch.zeros(sum(words), dtype=torch.int32, device="cuda")
    cnt = torch.zeros(len(tab), dtype=torch.int64, device="cuda")
    def call():
        _lib.call("fvv_carve", _lib.host_ptr(ds.cams), ctypes.c_int(ds.ncam), _lib.dev_ptr(ds.bits),
                  _lib.host_ptr(ds.word_off), _lib.host_ptr(tab), ctypes.c_int(len(tab)),
                  _lib.host_ptr(off), ctypes.c_int(1), _lib.dev_ptr(bits), _lib.dev_ptr(cnt),
                  _lib.dev_ptr(ws), ctypes.c_size_t(wsb), stream_handle())
    for _ in range(3): call()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(20): call()
    b.record(); torch.cuda.synchronize()
    aff = (96 * 128 * 64 + 255) & ~255
    st = ws[aff:aff + 24].view(torch.int64).tolist()
    cells = 16 * 135 * 8 * 2 * 4
    deferred = int(ws[wsb - (1 + 2 * (1 << 20)) * 8:wsb - 2 * (1 << 20) * 8].view(torch.int64).item())
    T = 16 if max(int(np.prod(g["dims"])) for g in tab) >= 4 << 20 else 8
    ntiles = sum(((int(g["dims"][0]) + T - 1) // T) * ((int(g["dims"][1]) + T - 1) // T) * ((int(g["dims"][2]) + T - 1) // T) for g in tab)
    live = ntiles - st[0]
    print(f"  tiles {ntiles}, culled {st[0]}, per live tile: fg cams {st[1] / max(live, 1):.2f}, mixed {st[2] / max(live, 1):.2f}")
    print(f"{name}: {sum(nvox)} voxels, {int(cnt.sum())} ON, deferred {deferred}, "
          f"{a.elapsed_time(b) / 20 * 1e3:.1f} us/launch pair")
