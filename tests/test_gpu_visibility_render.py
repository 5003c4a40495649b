"""GPU parity for D-1 / D-2 / E and the full run_frame: depth images,
triangle ids, visibility flags, rendered colours and source maps equal the
reference's golden outputs and the CPU oracle bit for bit."""

import ctypes
import json

import numpy as np
import pytest

import golden_io as G
import oracle as O

pytestmark = pytest.mark.gpu


def test_raster_golden_ties_winding_big_triangles(gpu):
    from paper_1903_11785_b200.mesh import TriangleMesh
    from paper_1903_11785_b200.visibility import classify_visibility, depth_image, rasterize

    z = G.load("raster")
    cam = G.camera(z, "cam")
    mesh = TriangleMesh(z["verts"], z["tris"])
    res = rasterize(mesh, cam)
    assert np.array_equal(res.depth, z["depth"])
    assert np.array_equal(res.tri_id, z["tri_id"])
    assert np.array_equal(classify_visibility(mesh, cam, res.depth, 50.0), z["vis"])
    one = TriangleMesh(z["one_verts"], [[0, 1, 2]])  # one triangle: numpy gemv centroid order
    assert np.array_equal(classify_visibility(one, cam, depth_image(one, cam), 10.0), z["one_vis"])
    empty = rasterize(TriangleMesh.empty(), cam)
    assert np.all(np.isinf(empty.depth)) and np.all(empty.tri_id == -1)


def test_visibility_maps_golden(gpu):
    from paper_1903_11785_b200.mesh import TriangleMesh
    from paper_1903_11785_b200.visibility import rasterize, visibility_maps

    z = G.load("spheres")
    rig = G.rig(z)
    mesh = TriangleMesh(z["vis_verts"], z["vis_tris"])
    depths, vis = visibility_maps(mesh, rig, t_v=150.0)
    assert np.array_equal(depths[rig[0].id], z["vis_depth0"])
    for i, c in enumerate(rig):
        assert np.array_equal(vis[c.id], G.unpack(z["vis_flags"][i], mesh.num_triangles)), c.id
    res = rasterize(mesh, rig[5])
    assert np.array_equal(res.depth, z["raster5_depth"])
    assert np.array_equal(res.tri_id, z["raster5_tri_id"])


@pytest.mark.parametrize("seed", range(3))
def test_raster_random_meshes_vs_oracle(gpu, seed):
    """Random cameras (incl. skew) and meshes mixing tiny, huge, behind-camera
    and sliver triangles; exact depth ties from duplicated triangles."""
    from paper_1903_11785_b200.camera import CameraModel
    from paper_1903_11785_b200.mesh import TriangleMesh
    from paper_1903_11785_b200.synthetic import look_at_camera
    from paper_1903_11785_b200.visibility import classify_visibility, rasterize

    rng = np.random.default_rng(seed)
    base = look_at_camera(0, rng.uniform([-3000, -3000, 800], [3000, 3000, 2500]),
                          (0, 0, 500), int(rng.integers(150, 420)), int(rng.integers(100, 300)),
                          float(rng.uniform(150, 500)))
    cam = CameraModel.from_dict(dict(base.to_dict(), skew=float(rng.normal(0, 0.02))))
    verts = rng.uniform([-900, -900, 0], [900, 900, 1200], (600, 3))
    small = np.repeat(rng.uniform([-900, -900, 0], [900, 900, 1200], (300, 1, 3)), 3, axis=1) + \
        rng.normal(0, 15, (300, 3, 3))
    verts = np.vstack([verts, small.reshape(-1, 3)])
    tris = np.vstack([rng.integers(0, 600, (150, 3)),
                      600 + np.arange(900).reshape(300, 3)]).astype(np.int32)
    tris = np.vstack([tris, tris[:20]])  # duplicates: exact depth ties
    mesh = TriangleMesh(verts, tris)
    res = rasterize(mesh, cam)
    depth, tid = O.rasterize(verts, tris, cam)
    assert np.array_equal(res.depth, depth)
    assert np.array_equal(res.tri_id, tid)
    assert np.array_equal(classify_visibility(mesh, cam, depth, 40.0),
                          O.classify(verts, tris, cam, depth, 40.0))


def test_classify_centroids_on_pixel_rounding_ties(gpu):
    """Centroids projecting exactly onto (and a few ulps either side of) the
    half-pixel rounding boundaries and the frustum edges: the visibility
    kernel's reciprocal fast path must fall back to the exact divisions there
    (np.rint ties to even)."""
    from paper_1903_11785_b200.camera import CameraModel
    from paper_1903_11785_b200.mesh import TriangleMesh
    from paper_1903_11785_b200.visibility import classify_visibility

    W, H = 64, 48
    cam = CameraModel.from_dict(dict(id=0, image_size=[W, H], fx=1.0, fy=1.0, cx=0.0, cy=0.0,
                                     skew=0.0, rotation=np.eye(3).tolist(),
                                     translation=[0.0, 0.0, 0.0]))
    rng = np.random.default_rng(11)
    n = 4000
    Z = rng.integers(500, 3000, n).astype(np.float64)
    ku = rng.integers(-2, W + 1, n) + 0.5
    kv = rng.integers(-2, H + 1, n) + 0.5
    X, Y = ku * Z, kv * Z  # u = X / Z = ku exactly: a rounding tie
    for arr in (X, Y):  # perturb some by a few ulps either way
        steps = rng.integers(-3, 4, n)
        for i in np.nonzero(steps)[0]:
            for _ in range(abs(int(steps[i]))):
                arr[i] = np.nextafter(arr[i], np.inf if steps[i] > 0 else -np.inf)
    verts = np.repeat(np.stack([X, Y, Z], axis=1), 3, axis=0)  # centroid == the point
    tris = np.arange(3 * n, dtype=np.int32).reshape(n, 3)
    depth = rng.uniform(400, 3100, (H, W))
    mesh = TriangleMesh(verts, tris)
    got = classify_visibility(mesh, cam, depth, 25.0)
    ref = O.classify(verts, tris, cam, depth, 25.0)
    assert np.array_equal(got, ref)
    assert 0 < ref.sum() < n


@pytest.mark.parametrize("name", ["tiny_cli", "figures"])
def test_run_frame_and_render_golden(gpu, name):
    """run_frame (pipeline.py:115-220) + render_view (render.py:64-113) on the
    reference's golden frames: stats, per-ROI meshes, visibility of every
    camera, camera-0 depth, rendered colours and source ids."""
    from paper_1903_11785_b200.pipeline import PipelineConfig, run_frame
    from paper_1903_11785_b200.render import render_view

    z = G.load(name)
    rig, sils = G.rig(z), G.sils(z)
    cfg_d = json.loads(str(z["cfg"]))
    cfg_d["t_large"] = float("inf") if cfg_d["t_large"] is None else cfg_d["t_large"]
    cfg = PipelineConfig(**{k: (tuple(v) if isinstance(v, list) else v) for k, v in cfg_d.items()})
    frames = G.frames(z, rig)
    bundle = run_frame(cfg, rig, frames, sils=sils, keep_depths=True)
    assert bundle.stats == json.loads(str(z["stats"]))
    for i, m in enumerate(bundle.meshes):
        assert np.array_equal(m.vertices, z[f"mesh{i}_verts"])
        assert np.array_equal(m.triangles, z[f"mesh{i}_tris"])
    merged = bundle.merged_mesh
    assert np.array_equal(merged.vertices, z["merged_verts"])
    assert np.array_equal(merged.triangles, z["merged_tris"])
    assert np.array_equal(merged.object_ids, z["merged_oids"])
    for i, c in enumerate(rig):
        assert np.array_equal(bundle.visibility[c.id], G.unpack(z["vis"][i], merged.num_triangles))
    assert np.array_equal(bundle.depths[rig[0].id], z["depth0"])
    assert set(bundle.timings.to_dict()) == {"sparse_carve", "noise_filter_roi", "dense_carve",
                                             "polygonize", "depth_images", "visibility"}
    virtual = G.camera(z, "virtual")
    img = render_view(merged, rig, frames, bundle.visibility, virtual)
    assert np.array_equal(img.source, z["render_source"])
    assert np.array_equal(img.color, z["render_color"])  # bit-exact (north_star allows 1/255)
    assert np.array_equal(img.covered, z["virtual_tri_id"] >= 0)


def test_render_vs_oracle_distorted_sources(gpu):
    """render_view with distorted/skewed source cameras vs the oracle."""
    from paper_1903_11785_b200.camera import CameraModel, CameraRig
    from paper_1903_11785_b200.pipeline import PipelineConfig, run_frame
    from paper_1903_11785_b200.render import render_view
    from paper_1903_11785_b200.synthetic import look_at_camera

    z = G.load("figures")
    rig0, sils = G.rig(z), G.sils(z)
    cams = []
    rng = np.random.default_rng(5)
    for c in rig0:
        d = c.to_dict()
        d["dist"] = [float(rng.normal(0, 0.02)), 0.0, float(rng.normal(0, 0.001)), 0.0, 0.0]
        d["skew"] = float(rng.normal(0, 0.005))
        cams.append(CameraModel.from_dict(d))
    rig = CameraRig(cams)
    cfg = PipelineConfig(stage_lo=(-2000, -2000, 0), stage_hi=(2000, 2000, 2000),
                         coarse_spacing=62.5, fine_spacing=31.25, t_small=3)
    frames = G.frames(z, rig0)
    bundle = run_frame(cfg, rig, frames, sils=sils)
    m = bundle.merged_mesh
    virtual = look_at_camera(50, (3900, -3500, 1500), (0, 0, 900), 300, 200, 260)
    img = render_view(m, rig, frames, bundle.visibility, virtual)
    color, source, covered = O.render_view(m.vertices, m.triangles, rig, frames,
                                           bundle.visibility, virtual)
    assert np.array_equal(img.source, source)
    assert np.array_equal(img.color, color)
    assert np.array_equal(img.covered, covered)


def test_render_reference_kats(gpu):
    """tests/test_render.py:24-55 ranking / source selection known answers."""
    from paper_1903_11785_b200.camera import CameraRig
    from paper_1903_11785_b200.render import rank_cameras, triangle_sources
    from paper_1903_11785_b200.synthetic import look_at_camera

    def cam_at(i, c):
        return look_at_camera(i, c, (0.0, 0.0, 0.0), 160, 120, 100.0)

    rig = CameraRig([cam_at(0, (4000, 0, 0)), cam_at(1, (2000, 0, 0)), cam_at(2, (0, 3000, 0))])
    assert rank_cameras(cam_at(99, (1900, 100, 0)), rig) == [1, 0, 2]
    rig = CameraRig([cam_at(5, (3000, 0, 0)), cam_at(2, (-3000, 0, 0))])
    assert rank_cameras(cam_at(99, (0, 3000, 0)), rig) == [2, 5]
    vis = {0: np.array([True, False, False]), 1: np.array([True, True, False]),
           2: np.array([True, True, True])}
    assert triangle_sources([0, 1, 2], vis, 3).tolist() == [0, 1, 2]
    assert triangle_sources([0, 1], {0: np.array([False]), 1: np.array([False])}, 1).tolist() == [-1]


def test_run_frame_empty_scene_and_errors(gpu):
    """tests/test_pipeline.py:99-122: empty scene -> valid empty bundle;
    stage errors carry the stage name."""
    from paper_1903_11785_b200.pipeline import PipelineConfig, StageError, run_frame

    z = G.load("spheres")
    rig = G.rig(z)
    cfg = PipelineConfig(stage_lo=(-1200, -1200, 0), stage_hi=(1200, 1200, 1200),
                         coarse_spacing=100.0, fine_spacing=50.0)
    empty = [np.zeros((c.image_height, c.image_width), dtype=bool) for c in rig]
    b = run_frame(cfg, rig, {c.id: None for c in rig}, sils=empty)
    assert b.stats["components"] == 0 and b.stats["triangles"] == 0 and b.meshes == []
    assert all(len(v) == 0 for v in b.visibility.values())
    with pytest.raises(StageError, match="silhouette"):
        run_frame(cfg, rig, {})
    bad = [np.ones((4, 4), dtype=bool) for _ in rig]
    with pytest.raises(StageError) as ei:
        run_frame(cfg, rig, {}, sils=bad)
    assert "B-1" in str(ei.value)


def test_run_sequence_matches_golden_frames(gpu):
    """pipeline.run_sequence (overlapped uploads; pinned colour frames sampled
    in place, pageable ones uploaded) returns the same bundles and images as the
    reference for a sequence mixing the two golden scenes' inputs."""
    import torch

    from paper_1903_11785_b200.pipeline import PipelineConfig, run_sequence

    z = G.load("figures")
    rig, sils = G.rig(z), G.sils(z)
    cfg_d = json.loads(str(z["cfg"]))
    cfg_d["t_large"] = float("inf")
    cfg = PipelineConfig(**{k: (tuple(v) if isinstance(v, list) else v) for k, v in cfg_d.items()})
    frames = {c.id: torch.from_numpy(z["frames"][i]).pin_memory() for i, c in enumerate(rig)}
    masks = torch.from_numpy(np.stack(sils).astype(np.uint8)).pin_memory()
    virtual = G.camera(z, "virtual")
    np_frames = {c.id: z["frames"][i] for i, c in enumerate(rig)}  # pageable: uploaded
    from paper_1903_11785_b200 import _lib

    lib = _lib.load()  # pinned frames are sampled in place, pageable ones uploaded
    assert all(lib.fvv_host_mapped(ctypes.c_void_p(f.data_ptr())) for f in frames.values())
    assert not any(lib.fvv_host_mapped(ctypes.c_void_p(f.ctypes.data)) for f in np_frames.values())
    out = list(run_sequence(cfg, rig, [frames, np_frames, frames], [masks, masks, sils],
                            virtual))
    assert len(out) == 3
    for bundle, img in out:
        assert bundle.stats == json.loads(str(z["stats"]))
        assert np.array_equal(bundle.merged_mesh.triangles, z["merged_tris"])
        assert np.array_equal(bundle.merged_mesh.vertices, z["merged_verts"])
        for i, c in enumerate(rig):
            assert np.array_equal(bundle.visibility[c.id],
                                  G.unpack(z["vis"][i], bundle.merged_mesh.num_triangles))
        assert np.array_equal(img.color, z["render_color"])
        assert np.array_equal(img.source, z["render_source"])


@pytest.mark.parametrize("width", [96, 4000])
def test_raster_fp32_filter_adversarial(gpu, width):
    """The FP32 candidate filter (raster_filter_kernel) against the exact
    float64 raster on tiny triangles built to sit on its decision boundaries:
    vertices on a 1/4-pixel lattice (edges through pixel centres: w == 0 and
    the top-left rule), slivers of near-zero area, vertices perturbed by a few
    ulps, triangles just outside the float extent, far from the image origin
    (4000 px wide: larger float rounding) and beyond the image border."""
    from paper_1903_11785_b200.camera import CameraModel
    from paper_1903_11785_b200.mesh import TriangleMesh
    from paper_1903_11785_b200.visibility import rasterize

    h = 48
    # R = I, t = 0, fx = fy = 1024, Z = 1024: u = X + cx exactly
    cam = CameraModel(0, width, h, 1024.0, 1024.0, 0.0, 0.0)
    rng = np.random.default_rng(width)
    n = 6000
    c = np.stack([rng.uniform(-2, width + 1, n), rng.uniform(-2, h + 1, n)], 1)
    uv = np.repeat(c[:, None, :], 3, axis=1)
    kind = rng.integers(0, 4, n)
    lat = np.round((uv + rng.uniform(-1.5, 1.5, (n, 3, 2))) * 4) / 4  # 1/4 px lattice
    uv = np.where(kind[:, None, None] == 0, lat, uv + rng.uniform(-1.2, 1.2, (n, 3, 2)))
    sl = kind == 1  # slivers: third vertex a hair off the first edge
    t = rng.uniform(0, 1, sl.sum())[:, None]
    uv[sl, 2] = uv[sl, 0] + t * (uv[sl, 1] - uv[sl, 0]) + rng.normal(0, 1e-4, (sl.sum(), 2))
    ulp = kind == 2  # lattice vertices nudged by a few ulps
    uv[ulp] = lat[ulp] + rng.integers(-3, 4, (ulp.sum(), 3, 2)) * np.spacing(lat[ulp] + 0.0)
    z = 1024.0 + np.round(rng.uniform(0, 64, (n, 3)))
    z[(kind == 0) | (kind == 2)] = 1024.0  # u = X exactly on the lattice
    verts = np.concatenate([uv * (z[..., None] / 1024.0), z[..., None]], axis=2).reshape(-1, 3)
    tris = np.arange(3 * n, dtype=np.int32).reshape(n, 3)
    mesh = TriangleMesh(verts, tris)
    res = rasterize(mesh, cam)
    depth, tid = O.rasterize(verts, tris, cam)
    assert np.isfinite(depth).sum() > 1000
    assert np.array_equal(res.depth, depth)
    assert np.array_equal(res.tri_id, tid)


def test_raster_pair_list_overflow_falls_back(gpu):
    """Every item of a warp list emitting three candidate pixels (more than
    the list's two per item) overflows the FP32 filter's pair lists: the
    sweep kernel then rasterises every item, with identical results."""
    from paper_1903_11785_b200.camera import CameraModel
    from paper_1903_11785_b200.mesh import TriangleMesh
    from paper_1903_11785_b200.visibility import rasterize

    cam = CameraModel(0, 160, 120, 1024.0, 1024.0, 0.0, 0.0)
    rng = np.random.default_rng(7)
    n = 4000
    base = np.stack([rng.integers(1, 150, n), rng.integers(1, 110, n)], 1) - 0.45
    uv = np.stack([base, base + [1.9, 0.0], base + [0.0, 1.9]], 1)  # 3 of 4 centres inside
    z = np.round(rng.uniform(1024.0, 1100.0, (n, 1)))  # ties between overlapping triangles
    z = np.repeat(z, 3, axis=1)
    verts = np.concatenate([uv * (z[..., None] / 1024.0), z[..., None]], axis=2).reshape(-1, 3)
    tris = np.arange(3 * n, dtype=np.int32).reshape(n, 3)
    res = rasterize(TriangleMesh(verts, tris), cam)
    depth, tid = O.rasterize(verts, tris, cam)
    assert np.isfinite(depth).sum() > 5000
    assert np.array_equal(res.depth, depth)
    assert np.array_equal(res.tri_id, tid)
