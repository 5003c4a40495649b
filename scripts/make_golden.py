"""Generate tests/golden/*.npz from the REFERENCE implementation itself.

Runs in the build container only (it imports /root/reference/pkg/src);
the fixtures it writes are committed and travel with the repo, so parity
tests on the GPU box never read /root/reference.

Every fixture stores the inputs (rig JSON, silhouettes, frames, grid
specs) and the reference's outputs for them. OpenBLAS is pinned to the
Haswell kernels (OPENBLAS_CORETYPE=Haswell) because the
reference's projection arithmetic goes through BLAS.

    python scripts/make_golden.py            # all fixtures
"""

from __future__ import annotations

import json
import os
import sys
import tempfile

if os.environ.get("OPENBLAS_CORETYPE") != "Haswell":
    env = dict(os.environ, OPENBLAS_CORETYPE="Haswell",
               NUMBA_CACHE_DIR=os.environ.get("NUMBA_CACHE_DIR", "/tmp/fvv_numba_cache"))
    os.execve(sys.executable, [sys.executable] + sys.argv, env)

import numpy as np  # noqa: E402

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
OUT = os.path.join(ROOT, "tests", "golden")

from freeview import camera as fcam  # noqa: E402
from freeview import hull as fhull  # noqa: E402
from freeview import mesh as fmesh  # noqa: E402
from freeview import pipeline as fpipe  # noqa: E402
from freeview import render as frender  # noqa: E402
from freeview import scenes as fscenes  # noqa: E402
from freeview import synthetic as fsyn  # noqa: E402
from freeview import visibility as fvis  # noqa: E402
from freeview.voxels import GridSpec, VoxelGrid  # noqa: E402

from paper_1903_11785_b200 import synthetic as oursyn  # noqa: E402  (ellipsoid figures)


def pack(b):
    return np.packbits(np.asarray(b, dtype=bool).reshape(-1), bitorder="little")


def rig_json(rig):
    return json.dumps(rig.to_dict())


def save(name, **arrays):
    os.makedirs(OUT, exist_ok=True)
    path = os.path.join(OUT, name + ".npz")
    np.savez_compressed(path, **arrays)
    print(f"{path}: {os.path.getsize(path) / 1e3:.1f} kB")


def spec_arr(spec):
    return np.array(list(spec.origin) + [spec.spacing] + list(spec.dims), dtype=np.float64)


def mesh_arrays(prefix, meshes):
    out = {}
    for i, m in enumerate(meshes):
        out[f"{prefix}{i}_verts"] = m.vertices
        out[f"{prefix}{i}_tris"] = m.triangles
        out[f"{prefix}{i}_oids"] = m.object_ids
    return out


def full_frame(name, rig, sils, frames, cfg, virtual, golden_stats=None):
    """run_frame + render_view through the reference's public API."""
    bundle = fpipe.run_frame(cfg, rig, frames, sils=sils, keep_depths=True)
    if golden_stats is not None:
        assert bundle.stats == golden_stats, (bundle.stats, golden_stats)
    spec = cfg.coarse_spec()
    coarse = fhull.carve(rig, sils, spec, cfg.min_views)
    lab = fhull.label_components(coarse, cfg.block_dims)
    _, lab_f = fhull.filter_noise(coarse, lab, cfg.noise_params)
    rois = fhull.extract_rois(lab_f, spec, cfg.roi_margin)
    fine = fhull.dense_carve(rig, sils, rois, cfg.fine_spacing, cfg.min_views)
    merged = bundle.merged_mesh
    arrays = dict(
        rig=rig_json(rig),
        cfg=json.dumps({k: (None if (k == "t_large" and np.isinf(v)) else v)
                        for k, v in cfg.__dict__.items()}),
        sils=np.stack([pack(s) for s in sils]),
        sil_shapes=np.array([s.shape for s in sils]),
        stats=json.dumps(bundle.stats),
        coarse_spec=spec_arr(spec),
        coarse_occ=pack(coarse.occ),
        labels=lab.labels,
        comps=np.array([[c.id, c.voxel_count, *c.bbox_min, *c.bbox_max] for c in lab.components],
                       dtype=np.int64).reshape(-1, 8),
        fcomps=np.array([c.id for c in lab_f.components], dtype=np.int64),
        rois=np.array([list(r.lo) + list(r.hi) + [r.component_id] for r in rois]).reshape(-1, 7),
        fine_specs=np.array([spec_arr(g.spec) for g in fine]).reshape(-1, 7),
        merged_verts=merged.vertices, merged_tris=merged.triangles,
        merged_oids=merged.object_ids,
        vis=np.stack([pack(bundle.visibility[c.id]) for c in rig]) if merged.num_triangles
        else np.zeros((len(rig), 0), np.uint8),
        depth0=bundle.depths[rig[0].id],
    )
    for i, g in enumerate(fine):
        arrays[f"fine{i}_occ"] = pack(g.occ)
    arrays.update(mesh_arrays("mesh", bundle.meshes))
    if frames is not None and virtual is not None:
        arrays["frames"] = np.stack([frames[c.id] for c in rig])
        arrays["virtual"] = json.dumps(virtual.to_dict())
        img = frender.render_view(merged, rig, frames, bundle.visibility, virtual)
        arrays["render_color"] = img.color
        arrays["render_source"] = img.source
        ras = fvis.rasterize(merged, virtual)
        arrays["virtual_depth"] = ras.depth
        arrays["virtual_tri_id"] = ras.tri_id
    save(name, **arrays)
    return bundle


def fixture_tiny_cli():
    """TINY_SPEC of tests/test_cli.py:11-23 through synth -> reconstruct; its
    stats must equal the reference's committed bundle manifest
    (pkg/frontend/tests/fixtures/bundle/manifest.json:29-38)."""
    spec = {
        "objects": [
            {"type": "sphere", "center": [-350, 0, 450], "radius": 250},
            {"type": "box", "lo": [300, -200, 200], "hi": [700, 200, 700],
             "color": [70, 110, 200]},
        ],
        "rig": {"n_cameras": 8, "target": [0, 0, 450], "ring_radius": 3500,
                "height": 1400, "width": 320, "image_height": 180, "focal": 260},
        "stage_lo": [-1000, -1000, 0],
        "stage_hi": [1000, 1000, 1000],
        "config": {"coarse_spacing": 80.0, "fine_spacing": 40.0, "t_small": 3},
        "noise_sigma": 1.5,
    }
    objects = fscenes.objects_from_spec(spec["objects"])
    rig = fscenes.default_rig_from_spec(spec["rig"])
    cfg = fpipe.PipelineConfig(stage_lo=tuple(spec["stage_lo"]), stage_hi=tuple(spec["stage_hi"]),
                               **spec["config"])
    _, frames, proposals, _, bg_frames = fscenes.generate_scene(
        objects, rig, cfg, noise_sigma=spec["noise_sigma"], seed=0)
    with tempfile.TemporaryDirectory() as d:
        fscenes.write_scene(d, rig, cfg, objects, frames, proposals, bg_frames)
        rig, cfg, frames, proposals, background = fscenes.read_scene(d)
    sils = fpipe.compute_silhouettes(cfg, rig, frames, proposals, background)
    man = json.load(open("/root/reference/pkg/frontend/tests/fixtures/bundle/manifest.json"))
    virtual = fsyn.look_at_camera(99, (2600, -2400, 1500), (0, 0, 450), 320, 180, 260)
    full_frame("tiny_cli", rig, sils, frames, cfg, virtual, golden_stats=man["stats"])


def fixture_figures():
    """C1-shaped scene with this repo's ellipsoid figures, scaled down so the
    reference's Python rasteriser finishes: 8 cams 320x240, 3 figures."""
    rig = fsyn.ring_rig(8, (0, 0, 900), 6000, 2000, 320, 240, 260)
    figs = oursyn.place_figures(3, (-1400, -1400), (1400, 1400), seed=3, t=0.2)
    ours_rig = oursyn.ring_rig(8, (0, 0, 900), 6000, 2000, 320, 240, 260)
    sils, frames = oursyn.render_scene(ours_rig, figs, shade=True, noise_sigma=1.0)
    cfg = fpipe.PipelineConfig(stage_lo=(-2000, -2000, 0), stage_hi=(2000, 2000, 2000),
                               coarse_spacing=62.5, fine_spacing=31.25, t_small=3)
    virtual = fsyn.look_at_camera(77, (4200, 3100, 1700), (0, 0, 900), 320, 240, 280)
    full_frame("figures", rig, sils, frames, cfg, virtual)


def fixture_spheres():
    """conftest small_rig + two spheres (tests/conftest.py:13-35): carve at
    several spacings incl. min_views, polygonize both modes, KAT grids."""
    rig = fsyn.ring_rig(12, target=(0, 0, 500), ring_radius=4000, height=1200, width=480,
                        image_height=270, focal=400)
    objs = [fsyn.Sphere(center=(-500, 0, 500), radius=350),
            fsyn.Sphere(center=(700, 0, 500), radius=300, color=np.array([60.0, 180.0, 90.0]))]
    sils = fsyn.scene_silhouettes(fsyn.SyntheticScene(rig=rig, objects=objs))
    arrays = dict(rig=rig_json(rig), sils=np.stack([pack(s) for s in sils]),
                  sil_shapes=np.array([s.shape for s in sils]))
    cases = [((-1200, -1200, 0), (1200, 1200, 1200), 60.0, 1),
             ((-1200, -1200, 0), (1200, 1200, 1200), 100.0, 12),
             ((-1200, -1200, 0), (1200, 1200, 1200), 100.0, 5),
             ((-1000, -500, 0), (1200, 500, 1000), 50.0, 1)]
    for i, (lo, hi, s, mv) in enumerate(cases):
        spec = GridSpec.from_aabb(lo, hi, s)
        g = fhull.carve(rig, sils, spec, min_views=mv)
        arrays[f"carve{i}_spec"] = spec_arr(spec)
        arrays[f"carve{i}_minv"] = np.array(mv)
        arrays[f"carve{i}_occ"] = pack(g.occ)
    # polygonize the 50 mm hull in both modes (mesh.py:275)
    spec = GridSpec.from_aabb((-1000, -500, 0), (1200, 500, 1000), 50.0)
    grid = fhull.carve(rig, sils, spec)
    for mode, iso in (("exact", 0.5), ("fixed", 0.25)):
        m, st = fmesh.polygonize(grid, rig, sils, mode=mode, fixed_isovalue=iso, object_id=4)
        arrays[f"poly_{mode}_verts"] = m.vertices
        arrays[f"poly_{mode}_tris"] = m.triangles
        arrays[f"poly_{mode}_stats"] = np.array([st.fallback_edges, st.inconsistent_starts])
    # single-voxel KAT grids (tests/test_mesh.py:160-184, 239-245)
    sv = GridSpec(origin=(0, 0, 0), spacing=10.0, dims=(3, 3, 3))
    occ = np.zeros(27, dtype=bool)
    occ[sv.linear_index(1, 1, 1)] = True
    allfg = [np.ones((c.image_height, c.image_width), dtype=bool) for c in rig]
    m, st = fmesh.polygonize(VoxelGrid(spec=sv, occ=occ), rig, allfg, mode="exact")
    arrays["single_exact_verts"], arrays["single_exact_tris"] = m.vertices, m.triangles
    m, _ = fmesh.polygonize(VoxelGrid(spec=sv, occ=occ), mode="fixed", fixed_isovalue=0.25)
    arrays["single_fixed_verts"], arrays["single_fixed_tris"] = m.vertices, m.triangles
    # visibility on the exact hull mesh, every camera (visibility.py:132-140)
    mesh, _ = fmesh.polygonize(grid, rig, sils, mode="exact")
    depths, vis = fvis.visibility_maps(mesh, rig, t_v=150.0)
    arrays["vis_verts"], arrays["vis_tris"] = mesh.vertices, mesh.triangles
    arrays["vis_flags"] = np.stack([pack(vis[c.id]) for c in rig])
    arrays["vis_depth0"] = depths[rig[0].id]
    ras = fvis.rasterize(mesh, rig[5])
    arrays["raster5_depth"], arrays["raster5_tri_id"] = ras.depth, ras.tri_id
    save("spheres", **arrays)


def random_camera(rng, cid, distorted=True, skew=True):
    w, h = int(rng.integers(160, 400)), int(rng.integers(120, 300))
    center = rng.uniform([-3000, -3000, 500], [3000, 3000, 2500])
    cam = fsyn.look_at_camera(cid, center, rng.uniform([-300, -300, 300], [300, 300, 700]), w, h,
                              float(rng.uniform(150, 400)))
    d = dict(cam.to_dict())
    if distorted:
        d["dist"] = [float(rng.normal(0, 0.08)), float(rng.normal(0, 0.02)),
                     float(rng.normal(0, 0.002)), float(rng.normal(0, 0.002)),
                     float(rng.normal(0, 0.005))]
    if skew:
        d["skew"] = float(rng.normal(0, 0.01))
    d["cx"] = float(d["cx"]) + float(rng.uniform(-3, 3))
    return fcam.CameraModel.from_dict(d)


def fixture_distorted():
    """Distorted, skewed random cameras: project (N=1 and batched), carve,
    exact isovalues against a sphere silhouette."""
    rng = np.random.default_rng(1234)
    cams = [random_camera(rng, i) for i in range(6)]
    rig = fcam.CameraRig(cams)
    sphere = fsyn.Sphere(center=(0, 0, 500), radius=450)
    sils = []
    for c in rig:  # silhouettes: analytic sphere seen through the undistorted twin camera
        zero = fcam.CameraModel.from_dict(dict(c.to_dict(), dist=[0.0] * 5, skew=0.0))
        sils.append(fsyn.analytic_silhouette(zero, [sphere]))
    pts = rng.uniform([-2000, -2000, -500], [2000, 2000, 2500], (1500, 3))
    arrays = dict(rig=rig_json(rig), pts=pts)
    arrays["sil_list"] = np.concatenate([pack(s) for s in sils])
    arrays["sil_shapes"] = np.array([s.shape for s in sils])
    for ci, c in enumerate(rig):
        px, z, inside = fcam.project(c, pts)
        arrays[f"proj{ci}_px"], arrays[f"proj{ci}_z"], arrays[f"proj{ci}_in"] = px, z, inside
        px1, z1, in1 = fcam.project(c, pts[ci])  # single point: gemv order
        arrays[f"proj{ci}_single"] = np.array([px1[0], px1[1], z1, float(in1)])
        px, z, inside = fcam.project(c, pts, use_distortion=False)
        arrays[f"projnd{ci}_px"] = px
    spec = GridSpec.from_aabb((-900, -900, 0), (900, 900, 1100), 45.0)
    arrays["carve_spec"] = spec_arr(spec)
    grid = fhull.carve(rig, sils, spec)
    arrays["carve_occ"] = pack(grid.occ)
    m, st = fmesh.polygonize(grid, rig, sils, mode="exact", object_id=2)
    arrays["poly_verts"], arrays["poly_tris"] = m.vertices, m.triangles
    arrays["poly_stats"] = np.array([st.fallback_edges, st.inconsistent_starts])
    save("distorted", **arrays)


def fixture_ccl():
    """Random grids at the densities of tests/test_hull.py:152-157 plus the
    hand KATs of tests/test_hull.py:119-149."""
    rng = np.random.default_rng(7)
    arrays = {}
    cases = [((24, 24, 24), 0.05), ((24, 24, 24), 0.2), ((24, 24, 24), 0.5), ((17, 9, 31), 0.3),
             ((40, 3, 5), 0.45), ((1, 1, 50), 0.6), ((33, 33, 1), 0.35), ((64, 48, 40), 0.08)]
    for i, (dims, dens) in enumerate(cases):
        spec = GridSpec(origin=(0, 0, 0), spacing=10.0, dims=dims)
        occ = rng.random(spec.num_voxels) < dens
        lab = fhull.label_components(VoxelGrid(spec=spec, occ=occ), block_dims=(8, 8, 8))
        arrays[f"g{i}_dims"] = np.array(dims)
        arrays[f"g{i}_occ"] = pack(occ)
        arrays[f"g{i}_labels"] = lab.labels
        arrays[f"g{i}_comps"] = np.array(
            [[c.id, c.voxel_count, *c.bbox_min, *c.bbox_max] for c in lab.components],
            dtype=np.int64).reshape(-1, 8)
        fg, fl = fhull.filter_noise(VoxelGrid(spec=spec, occ=occ), lab,
                                    fhull.NoiseFilterParams(t_small=3, t_large=40))
        arrays[f"g{i}_flabels"] = fl.labels
    save("ccl", **arrays)


def fixture_raster():
    """Random triangles (tests/test_visibility.py:97-135) with ties, shared
    edges, reversed winding and behind-camera geometry."""
    cam = fcam.CameraModel(id=0, image_width=160, image_height=120, fx=100.0, fy=100.0,
                           cx=79.5, cy=59.5)
    rng = np.random.default_rng(11)

    def screen(pix, z):
        return np.array([[(u - cam.cx) * z / cam.fx, (v - cam.cy) * z / cam.fy, z]
                         for u, v in pix])

    tris = [screen(rng.uniform([15, 15], [145, 105], (3, 2)), float(rng.uniform(1500, 9000)))
            + rng.uniform(-200, 200, (3, 1)) * np.array([0.0, 0.0, 1.0]) for _ in range(60)]
    base = screen([(20, 20), (120, 20), (70, 100)], 4000.0)
    tris += [base, base, base[[0, 2, 1]]]  # exact ties, reversed winding
    quad = screen([(30, 30), (130, 30), (130, 90), (30, 90)], 2000.0)
    tris += [quad[[0, 1, 2]], quad[[0, 2, 3]]]  # shared edge
    tris += [screen([(10, 10), (60, 10), (30, 50)], -1000.0)]  # behind the camera
    tris += [screen([(70.5, 30.5), (90.5, 30.5), (80.5, 50.5)], 3000.0)]  # half-pixel vertices
    verts = np.vstack(tris)
    tri_idx = np.arange(len(verts)).reshape(-1, 3)
    mesh = fmesh.TriangleMesh(verts, tri_idx)
    ras = fvis.rasterize(mesh, cam)
    vis = fvis.classify_visibility(mesh, cam, ras.depth, t_v=50.0)
    one = fmesh.TriangleMesh(tris[0], [[0, 1, 2]])
    vis1 = fvis.classify_visibility(one, cam, fvis.depth_image(one, cam), t_v=10.0)
    save("raster", cam=json.dumps(cam.to_dict()), verts=verts, tris=tri_idx, depth=ras.depth,
         tri_id=ras.tri_id, vis=vis, one_verts=tris[0], one_vis=vis1)


def fixture_bundle():
    """write_bundle (bundle.py:77-136, meshio.py, imgio.py) of the TINY_SPEC
    frame: sha256 of every file except the non-deterministic timings.json."""
    import hashlib

    from freeview.bundle import write_bundle

    z = np.load(os.path.join(OUT, "tiny_cli.npz"))
    rig = fcam.CameraRig([fcam.CameraModel.from_dict(d)
                          for d in json.loads(str(z["rig"]))["cameras"]])
    shapes = z["sil_shapes"]
    sils = [np.unpackbits(z["sils"][i], bitorder="little")[:h * w].astype(bool).reshape(h, w)
            for i, (h, w) in enumerate(shapes)]
    d = json.loads(str(z["cfg"]))
    d["t_large"] = float("inf") if d["t_large"] is None else d["t_large"]
    cfg = fpipe.PipelineConfig(**{k: (tuple(v) if isinstance(v, list) else v) for k, v in d.items()})
    frames = {c.id: z["frames"][i] for i, c in enumerate(rig)}
    bundle = fpipe.run_frame(cfg, rig, frames, sils=sils, frame_id=7, keep_depths=True)
    hashes = {}
    with tempfile.TemporaryDirectory() as tmp:
        write_bundle(bundle, tmp, export_depth=True)
        for root, _, files in os.walk(tmp):
            for fn in files:
                rel = os.path.relpath(os.path.join(root, fn), tmp)
                if rel == "timings.json":
                    continue
                with open(os.path.join(root, fn), "rb") as fh:
                    hashes[rel] = hashlib.sha256(fh.read()).hexdigest()
    with open(os.path.join(OUT, "bundle_sha256.json"), "w") as fh:
        json.dump(dict(sorted(hashes.items())), fh, indent=1)
        fh.write("\n")
    print(f"bundle hashes: {len(hashes)} files")


def fixture_silhouette():
    """silhouette.py (distance_map, build_background, extract_silhouette) and
    run_frame's proposal path (pipeline.py:104-112, 130-137) on a small
    scene generated by the reference's own scenes.generate_scene."""
    from freeview import silhouette as fsil

    objects = fscenes.objects_from_spec([
        {"type": "sphere", "center": [-250, 0, 450], "radius": 220},
        {"type": "box", "lo": [150, -150, 250], "hi": [450, 150, 650]},
    ])
    rig = fscenes.default_rig_from_spec({"n_cameras": 4, "target": [0, 0, 450],
                                         "ring_radius": 3200, "height": 1200, "width": 128,
                                         "image_height": 96, "focal": 110})
    cfg = fpipe.PipelineConfig(stage_lo=(-1000, -1000, 0), stage_hi=(1000, 1000, 1000),
                               coarse_spacing=80.0, fine_spacing=40.0, t_small=3)
    _, frames, proposals, _, bg_frames = fscenes.generate_scene(objects, rig, cfg,
                                                                noise_sigma=2.0, seed=5)
    arrays = dict(rig=rig_json(rig), cfg=json.dumps({k: (None if (k == "t_large" and np.isinf(v))
                                                         else v) for k, v in cfg.__dict__.items()}))
    for i, c in enumerate(rig):
        bg = fsil.build_background(bg_frames[c.id])
        dm = fsil.distance_map(proposals[c.id])
        sil = fsil.extract_silhouette(frames[c.id], bg, dm, cfg.adaptive_params)
        arrays[f"frame{i}"] = frames[c.id]
        arrays[f"prop{i}"] = pack(proposals[c.id])
        arrays[f"bgframes{i}"] = np.stack(bg_frames[c.id])
        arrays[f"dm{i}"] = dm
        arrays[f"sil{i}"] = pack(sil)
        if i < 2:
            arrays[f"bgmean{i}"], arrays[f"bgstd{i}"] = bg.mean, bg.std
    # edge cases: empty proposal, full proposal, single pixel
    arrays["dm_empty"] = fsil.distance_map(np.zeros((5, 7), dtype=bool))
    one = np.zeros((40, 50), dtype=bool)
    one[3, 47] = True
    arrays["dm_one"] = fsil.distance_map(one)
    rng = np.random.default_rng(9)
    rnd = rng.random((61, 83)) < 0.03
    arrays["rnd_prop"] = pack(rnd)
    arrays["dm_rnd"] = fsil.distance_map(rnd)
    background = {c.id: fsil.build_background(bg_frames[c.id]) for c in rig}
    bundle = fpipe.run_frame(cfg, rig, frames, proposals=proposals, background=background)
    arrays["stats"] = json.dumps(bundle.stats)
    save("silhouette", **arrays)


def fixture_grid_dump():
    """voxels.save_grid files written by the reference: random, all-on,
    all-off, a 64^3 solid, ragged word tails, and a carved grid."""
    from freeview.voxels import save_grid

    rng = np.random.default_rng(11)
    cases = [((4, 5, 6), rng.random(120) < 0.3), ((3, 3, 3), np.ones(27, dtype=bool)),
             ((3, 3, 3), np.zeros(27, dtype=bool)), ((64, 64, 64), np.ones(64 ** 3, dtype=bool)),
             ((33, 1, 1), rng.random(33) < 0.5), ((31, 2, 3), rng.random(186) < 0.7),
             ((1, 1, 1), np.ones(1, dtype=bool))]
    z = np.load(os.path.join(OUT, "spheres.npz"))
    sp = z["carve3_spec"]
    dims = tuple(int(d) for d in sp[4:7])
    cases.append((dims, np.unpackbits(z["carve3_occ"], bitorder="little")[:int(np.prod(dims))]
                  .astype(bool)))
    arrays = {}
    with tempfile.TemporaryDirectory() as tmp:
        for i, (dims, occ) in enumerate(cases):
            spec = GridSpec(origin=(-10.0 + i, 5.0, 0.25 * i), spacing=25.0 + i, dims=dims)
            path = os.path.join(tmp, f"g{i}.bin")
            save_grid(VoxelGrid(spec=spec, occ=occ), path)
            arrays[f"g{i}_dims"] = np.array(dims, dtype=np.int64)
            arrays[f"g{i}_origin"] = spec.origin
            arrays[f"g{i}_spacing"] = np.float64(spec.spacing)
            arrays[f"g{i}_occ"] = pack(occ)
            arrays[f"g{i}_file"] = np.frombuffer(open(path, "rb").read(), dtype=np.uint8)
    save("grid_dump", **arrays)


def fixture_synth():
    """The reference's Sphere/Box scene generator (synthetic.py:165-243):
    silhouettes, noiseless and noisy frames, eroded proposals, on the
    TINY_SPEC objects seen by a small ring plus a skewed camera and a camera
    looking straight down a box face."""
    objs = [fsyn.Sphere(center=[-350, 0, 450], radius=250),
            fsyn.Box(lo=[300, -200, 200], hi=[700, 200, 700], color=[70, 110, 200]),
            fsyn.Sphere(center=[0, 400, 300], radius=120, color=[90, 200, 120])]
    rig = fsyn.ring_rig(4, [0, 0, 450], 3500, 1400, width=160, image_height=120, focal=140)
    cams = list(rig)
    skew = fcam.CameraModel(id=7, image_width=150, image_height=110, fx=150.0, fy=140.0,
                            cx=70.3, cy=52.1, skew=0.35, rotation=cams[1].rotation,
                            translation=cams[1].translation)
    down = fsyn.look_at_camera(9, [500.0, 0.0, 3000.0], [500.0, 0.0, 700.0], 128, 96, 300.0)
    cams += [skew, down]
    rig = fcam.CameraRig(cams)
    scene = fsyn.SyntheticScene(rig=rig, objects=objs)
    arrays = {"rig": np.array(rig_json(rig))}
    for i, cam in enumerate(cams):
        sil = fsyn.analytic_silhouette(cam, objs)
        arrays[f"sil{i}"] = pack(sil)
        arrays[f"frame{i}"] = fsyn.shade_frame(scene, cam, 0.0, 0)
        arrays[f"noisy{i}"] = fsyn.shade_frame(scene, cam, 1.5, 3)
        arrays[f"prop{i}"] = pack(fsyn.proposal_from_silhouette(sil, 3))
        arrays[f"prop1_{i}"] = pack(fsyn.proposal_from_silhouette(sil, 1))
    save("synth", **arrays)


if __name__ == "__main__":
    which = sys.argv[1:] or ["tiny_cli", "spheres", "distorted", "ccl", "raster", "figures",
                             "silhouette", "bundle", "grid_dump", "synth"]
    for w in which:
        globals()[f"fixture_{w}"]()
