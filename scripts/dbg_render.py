import sys, json; sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import numpy as np, golden_io as G, torch
from paper_1903_11785_b200.pipeline import PipelineConfig, run_frame
from paper_1903_11785_b200 import render as R
z = G.load("tiny_cli"); rig, sils = G.rig(z), G.sils(z)
cfg_d = json.loads(str(z["cfg"])); cfg_d["t_large"] = float("inf")
cfg = PipelineConfig(**{k: (tuple(v) if isinstance(v, list) else v) for k, v in cfg_d.items()})
frames = G.frames(z, rig)
b = run_frame(cfg, rig, frames, sils=sils)
torch.cuda.synchronize(); print("frame ok", b.stats)
m = b.merged_mesh
virtual = G.camera(z, "virtual")
verts, tris = m.device_arrays()
print("verts", verts.shape, "tris", tris.shape, "tri max", int(tris.max()), "nt", m.num_triangles)
dev = verts.device
bits, stride = R._vis_bits_from_dict(b.visibility, list(rig), m.num_triangles, dev); torch.cuda.synchronize(); print("bits ok", bits.shape, stride)
planes = R.raster_planes(verts, tris, [virtual], want_ids=True); torch.cuda.synchronize(); print("raster ok")
src = R.sources_device(R.rank_cameras(virtual, rig), list(rig), bits, stride, m.num_triangles); torch.cuda.synchronize(); print("sources ok", src[:10])
fbuf, foff = R.frames_device(list(rig), frames, dev); torch.cuda.synchronize(); print("frames ok", fbuf.shape, foff)
img = R.render_view(m, rig, frames, b.visibility, virtual); print("render ok")
