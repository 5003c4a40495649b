"""GPU parity: projection and B-1/B-3 carving through libfvv.so against the
reference's golden outputs (tests/golden) and the CPU oracle, bit-exact."""

import numpy as np
import pytest

import golden_io as G
import oracle as O

pytestmark = pytest.mark.gpu


def test_project_matches_reference_bitwise(gpu):
    from paper_1903_11785_b200.camera import project

    z = G.load("distorted")
    rig = G.rig(z)
    pts = z["pts"]
    for ci, c in enumerate(rig):
        px, zz, inside = project(c, pts)
        assert np.array_equal(px, z[f"proj{ci}_px"])
        assert np.array_equal(zz, z[f"proj{ci}_z"])
        assert np.array_equal(inside, z[f"proj{ci}_in"])
        p1, z1, i1 = project(c, pts[ci])  # single point: reference's gemv order
        assert np.array_equal(np.array([p1[0], p1[1], z1, float(i1)]), z[f"proj{ci}_single"])
        px, _, _ = project(c, pts, use_distortion=False)
        assert np.array_equal(px, z[f"projnd{ci}_px"])


def test_carve_matches_reference_golden(gpu):
    from paper_1903_11785_b200.hull import carve

    z = G.load("spheres")
    rig, sils = G.rig(z), G.sils(z)
    for i in range(4):
        sp = G.spec(z[f"carve{i}_spec"])
        grid = carve(rig, sils, sp, min_views=int(z[f"carve{i}_minv"]))
        ref = G.unpack(z[f"carve{i}_occ"], sp.num_voxels)
        assert np.array_equal(grid.occ, ref), i
        assert grid.occupied_count == int(ref.sum())
    z = G.load("distorted")
    rig, sils = G.rig(z), G.sils(z)
    sp = G.spec(z["carve_spec"])
    assert np.array_equal(carve(rig, sils, sp).occ, G.unpack(z["carve_occ"], sp.num_voxels))


def test_dense_carve_batch_matches_golden_fine_grids(gpu):
    from paper_1903_11785_b200.hull import Roi, dense_carve

    for name in ("tiny_cli", "figures"):
        z = G.load(name)
        rig, sils = G.rig(z), G.sils(z)
        rois = [Roi(r[:3], r[3:6], int(r[6])) for r in z["rois"]]
        fine = float(z["fine_specs"][0][3])
        grids = dense_carve(rig, sils, rois, fine)
        assert len(grids) == len(rois)
        for i, g in enumerate(grids):
            assert np.array_equal(np.r_[g.spec.origin, g.spec.spacing, g.spec.dims],
                                  z["fine_specs"][i])
            assert np.array_equal(g.occ, G.unpack(z[f"fine{i}_occ"], g.spec.num_voxels)), (name, i)


def test_carve_edge_cases_vs_oracle(gpu):
    """Single-voxel chunk (gemv order), 1-voxel grids, ragged word tails,
    min_views > #cams, all-background and all-foreground silhouettes."""
    from paper_1903_11785_b200.hull import carve
    from paper_1903_11785_b200.voxels import GridSpec

    z = G.load("distorted")
    rig, sils = G.rig(z), G.sils(z)
    allfg = [np.ones_like(s) for s in sils]
    allbg = [np.zeros_like(s) for s in sils]
    specs = [
        GridSpec(origin=(-40.0, -25.0, 480.0), spacing=13.0, dims=(1, 1, 1)),
        GridSpec(origin=(-900.0, -900.0, 0.0), spacing=45.0, dims=(31, 17, 5)),
        GridSpec(origin=(-700.0, -600.0, 10.0), spacing=7.0, dims=(1 << 10, 1 << 10, 1)),  # 2^20
        GridSpec(origin=(-700.0, -600.0, 10.0), spacing=1.0, dims=(1, 1, (1 << 20) + 1)),
    ]
    for sp in specs:
        for s, mv in ((sils, 1), (allfg, 1), (allfg, 3), (allbg, 1), (sils, 7)):
            ref = O.carve(rig, s, sp.origin, sp.spacing, sp.dims, mv)
            got = carve(rig, s, sp, min_views=mv).occ
            assert np.array_equal(got, ref), (sp.dims, mv)


def test_carve_errors_match_reference_messages(gpu):
    from paper_1903_11785_b200.hull import carve
    from paper_1903_11785_b200.voxels import GridSpec

    z = G.load("spheres")
    rig = G.rig(z)
    sp = GridSpec.from_aabb((-1200, -1200, 0), (1200, 1200, 1200), 100.0)
    with pytest.raises(ValueError, match="silhouette shape"):
        carve(rig, [np.ones((8, 8), dtype=bool) for _ in rig], sp)
    with pytest.raises(ValueError, match="silhouettes for"):
        carve(rig, [], sp)


def _comp_rows(comps):
    return np.array([[c.id, c.voxel_count, *c.bbox_min, *c.bbox_max] for c in comps],
                    dtype=np.int64).reshape(-1, 8)


def test_ccl_matches_reference_golden(gpu):
    from paper_1903_11785_b200.hull import NoiseFilterParams, filter_noise, label_components
    from paper_1903_11785_b200.voxels import GridSpec, VoxelGrid

    z = G.load("ccl")
    for i in range(8):
        dims = tuple(int(d) for d in z[f"g{i}_dims"])
        spec = GridSpec(origin=(0, 0, 0), spacing=10.0, dims=dims)
        grid = VoxelGrid(spec, G.unpack(z[f"g{i}_occ"], spec.num_voxels))
        lab = label_components(grid)
        assert np.array_equal(_comp_rows(lab.components), z[f"g{i}_comps"]), i
        assert np.array_equal(lab.labels, z[f"g{i}_labels"]), i
        fgrid, flab = filter_noise(grid, lab, NoiseFilterParams(t_small=3, t_large=40))
        assert np.array_equal(flab.labels, z[f"g{i}_flabels"]), i
        assert np.array_equal(fgrid.occ, z[f"g{i}_flabels"] > 0), i
        assert fgrid.occupied_count == int((z[f"g{i}_flabels"] > 0).sum())


@pytest.mark.parametrize("seed", range(6))
def test_ccl_random_vs_oracle(gpu, seed):
    from paper_1903_11785_b200.hull import label_components
    from paper_1903_11785_b200.voxels import GridSpec, VoxelGrid

    rng = np.random.default_rng(100 + seed)
    for _ in range(5):
        dims = tuple(int(d) for d in rng.integers(1, 70, 3))
        dens = float(rng.choice([0.02, 0.1, 0.3, 0.6, 0.9]))
        spec = GridSpec(origin=(0, 0, 0), spacing=1.0, dims=dims)
        occ = rng.random(spec.num_voxels) < dens
        lab = label_components(VoxelGrid(spec, occ))
        ref_labels, ref_comps = O.label(occ, dims)
        assert np.array_equal(lab.labels, ref_labels), (dims, dens)
        assert np.array_equal(_comp_rows(lab.components), _comp_rows(ref_comps))


def test_ccl_reference_kats(gpu):
    """tests/test_hull.py:119-149 known answers."""
    from paper_1903_11785_b200.hull import label_components
    from paper_1903_11785_b200.voxels import GridSpec, VoxelGrid

    spec = GridSpec(origin=(0, 0, 0), spacing=1.0, dims=(4, 4, 4))
    lab = label_components(VoxelGrid(spec, np.zeros(64, dtype=bool)))
    assert lab.components == [] and not lab.labels.any()
    spec = GridSpec(origin=(0, 0, 0), spacing=1.0, dims=(3, 3, 3))
    occ = np.zeros(27, dtype=bool)
    occ[spec.linear_index(0, 0, 0)] = occ[spec.linear_index(1, 1, 1)] = True
    lab = label_components(VoxelGrid(spec, occ))
    assert len(lab.components) == 1 and lab.components[0].voxel_count == 2
    spec = GridSpec(origin=(0, 0, 0), spacing=1.0, dims=(5, 1, 1))
    lab = label_components(VoxelGrid(spec, np.array([True, False, True, True, False])))
    assert [c.voxel_count for c in lab.components] == [1, 2]
    assert lab.labels[0] == 1 and lab.labels[2] == 2
    spec = GridSpec(origin=(0, 0, 0), spacing=1.0, dims=(6, 6, 6))
    occ = np.zeros(spec.num_voxels, dtype=bool)
    for ijk in [(1, 2, 3), (2, 2, 3), (2, 3, 4)]:
        occ[spec.linear_index(*ijk)] = True
    lab = label_components(VoxelGrid(spec, occ))
    assert lab.components[0].bbox_min == (1, 2, 3) and lab.components[0].bbox_max == (2, 3, 4)
    with pytest.raises(ValueError):
        label_components(VoxelGrid(spec, occ), block_dims=(0, 1, 1))


def test_coarse_labels_of_full_frames(gpu):
    from paper_1903_11785_b200.hull import carve, label_components

    for name in ("tiny_cli", "figures"):
        z = G.load(name)
        rig, sils = G.rig(z), G.sils(z)
        spec = G.spec(z["coarse_spec"])
        grid = carve(rig, sils, spec)
        lab = label_components(grid)
        assert np.array_equal(_comp_rows(lab.components), z["comps"])
        assert np.array_equal(lab.labels, z["labels"])


def test_carve_fp32_filter_on_exact_half_pixels(gpu):
    """Voxel centres that project exactly onto pixel boundaries (u, v =
    k + 0.5) and onto the image borders: the certified float32 filter must
    hand every such test to the float64 chain (round-half-to-even)."""
    from paper_1903_11785_b200.camera import CameraModel, CameraRig
    from paper_1903_11785_b200.hull import carve
    from paper_1903_11785_b200.voxels import GridSpec

    rng = np.random.default_rng(3)
    cams = [CameraModel(id=0, image_width=200, image_height=100, fx=100.0, fy=100.0, cx=99.5,
                        cy=49.5),
            CameraModel(id=1, image_width=201, image_height=101, fx=50.0, fy=50.0, cx=100.0,
                        cy=50.0, skew=0.25)]
    rig = CameraRig(cams)
    sils = [rng.random((c.image_height, c.image_width)) < 0.5 for c in cams]
    for origin, spacing, dims in [((-1205.0, -605.0, 995.0), 10.0, (241, 121, 3)),
                                  ((-2010.0, -1010.0, 1990.0), 20.0, (202, 102, 2)),
                                  ((-40.0, -40.0, 2.0), 0.5, (160, 160, 4))]:
        spec = GridSpec(origin=origin, spacing=spacing, dims=dims)
        got = carve(rig, sils, spec).occ
        ref = O.carve(rig, sils, spec.origin, spec.spacing, spec.dims)
        assert np.array_equal(got, ref), origin
        assert got.any() and not got.all()


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_carve_tiles_random_rigs_vs_oracle(gpu, seed):
    """The tile-culled, certified-FP32 carve against the float64 oracle on
    random rigs: cameras close to and inside the grid (Z near / below 0,
    rectangles leaving the image), blocky silhouettes (whole tiles
    foreground or background), coarse (16^3 tiles) and fine (8^3) grids."""
    from paper_1903_11785_b200.camera import CameraModel, CameraRig
    from paper_1903_11785_b200.hull import carve
    from paper_1903_11785_b200.synthetic import look_at_camera
    from paper_1903_11785_b200.voxels import GridSpec

    rng = np.random.default_rng(100 + seed)
    cams = []
    for c in range(6):
        d = rng.uniform(400.0, 3000.0)
        ang = rng.uniform(0, 2 * np.pi)
        eye = (d * np.cos(ang), d * np.sin(ang), rng.uniform(-200.0, 1500.0))
        w, h = int(rng.integers(96, 200)), int(rng.integers(64, 160))
        cams.append(look_at_camera(c, eye, (rng.uniform(-200, 200), rng.uniform(-200, 200), 300.0),
                                   w, h, float(rng.uniform(60, 240))))
    rig = CameraRig(cams)
    sils = []
    for cam in cams:
        s = np.zeros((cam.image_height, cam.image_width), dtype=bool)
        for _ in range(4):  # blocky foreground
            y0, x0 = rng.integers(0, cam.image_height), rng.integers(0, cam.image_width)
            s[y0:y0 + rng.integers(5, 60), x0:x0 + rng.integers(5, 80)] = True
        s |= rng.random(s.shape) < 0.02
        sils.append(s)
    specs = [GridSpec(origin=(-2000.0, -1800.0, -300.0), spacing=20.0, dims=(200, 180, 120)),
             GridSpec(origin=(-600.0, -500.0, 0.0), spacing=7.5, dims=(90, 70, 60))]
    for sp in specs:
        for mv in (1, 2):
            ref = O.carve(rig, sils, sp.origin, sp.spacing, sp.dims, mv)
            got = carve(rig, sils, sp, min_views=mv).occ
            assert np.array_equal(got, ref), (seed, sp.dims, mv)


@pytest.mark.parametrize("dtype", ["float32", "int32", "float64"])
def test_non_bool_silhouettes_are_coerced_like_reference(gpu, dtype):
    """hull.py:68 casts every silhouette with np.asarray(sil, dtype=bool):
    a float / int mask with values other than 0/1 must carve like its bool
    form, whether handed over as numpy arrays, a stacked (N,H,W) torch
    tensor, or DeviceSilhouettes."""
    import torch

    from paper_1903_11785_b200._device import DeviceSilhouettes
    from paper_1903_11785_b200.hull import carve
    from paper_1903_11785_b200.pipeline import PipelineConfig, run_frame

    z = G.load("spheres")
    rig, sils = G.rig(z), G.sils(z)
    sp = G.spec(z["carve0_spec"])
    ref = carve(rig, sils, sp).occ
    scaled = [s.astype(dtype) * 0.75 if dtype != "int32" else s.astype(dtype) * 256
              for s in sils]
    assert np.array_equal(carve(rig, scaled, sp).occ, ref)
    stacked = torch.from_numpy(np.stack(scaled))
    assert np.array_equal(carve(rig, DeviceSilhouettes(rig, stacked), sp).occ, ref)
    cfg = PipelineConfig(stage_lo=tuple(sp.origin), stage_hi=tuple(
        sp.origin + sp.spacing * np.asarray(sp.dims)), coarse_spacing=sp.spacing,
        fine_spacing=sp.spacing / 2, t_small=3)
    frames = {c.id: None for c in rig}
    a = run_frame(cfg, rig, frames, sils=sils)
    b = run_frame(cfg, rig, frames, sils=stacked.cuda())
    assert a.stats == b.stats
    assert np.array_equal(a.merged_mesh.triangles, b.merged_mesh.triangles)


def test_ccl_separate_launches_match_oracle(gpu):
    """B-2 runs as one cooperative launch (ccl_fused_kernel); FVV_CCL_FUSED=0
    keeps the separate scan / union / scan / stats launches. Both numberings
    equal the oracle's (the separate path runs in a child process: the switch
    is read once per process)."""
    import os
    import subprocess
    import sys

    code = r'''
import sys, numpy as np
sys.path.insert(0, "tests")
import oracle as O
from paper_1903_11785_b200.hull import label_components
from paper_1903_11785_b200.voxels import GridSpec, VoxelGrid
rng = np.random.default_rng(7)
for _ in range(6):
    dims = tuple(int(d) for d in rng.integers(1, 60, 3))
    dens = float(rng.choice([0.05, 0.3, 0.7]))
    spec = GridSpec(origin=(0, 0, 0), spacing=1.0, dims=dims)
    occ = rng.random(spec.num_voxels) < dens
    lab = label_components(VoxelGrid(spec, occ))
    ref_labels, ref_comps = O.label(occ, dims)
    assert np.array_equal(lab.labels, ref_labels), (dims, dens)
    assert len(lab.components) == len(ref_comps)
print("ok")
'''
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, FVV_CCL_FUSED="0")
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stderr[-2000:]
