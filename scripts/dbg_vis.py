import sys; sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import numpy as np, golden_io as G, oracle as O
from paper_1903_11785_b200.mesh import TriangleMesh
from paper_1903_11785_b200.visibility import visibility_maps, classify_visibility, rasterize, depth_image
zr = G.load("raster"); cam = G.camera(zr, "cam")
m0 = TriangleMesh(zr["verts"], zr["tris"]); res = rasterize(m0, cam)
print("raster ok", np.array_equal(res.depth, zr["depth"]), np.array_equal(classify_visibility(m0, cam, res.depth, 50.0), zr["vis"]))
z = G.load("spheres"); rig = G.rig(z)
mesh = TriangleMesh(z["vis_verts"], z["vis_tris"])
for rep in range(3):
    depths, vis = visibility_maps(mesh, rig, t_v=150.0)
    for i, c in enumerate(rig):
        gold = G.unpack(z["vis_flags"][i], mesh.num_triangles)
        ref = O.classify(mesh.vertices, mesh.triangles, c, depths[c.id], 150.0)
        bad = np.flatnonzero(gold != vis[c.id])
        if len(bad): print(rep, i, "bad", len(bad), bad[:8], "ref-vs-gold", int((ref != gold).sum()), "depth eq", np.array_equal(depths[c.id], O.rasterize(mesh.vertices, mesh.triangles, c)[0]))
print("done")
