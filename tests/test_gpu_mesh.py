"""GPU parity for stage C (mesh.py): polygonize vertices/triangles bit-exact
against the reference's golden outputs and the CPU oracle, isovalue KATs
of tests/test_mesh.py, batched ROI meshing of full frames."""

import numpy as np
import pytest

import golden_io as G
import oracle as O

pytestmark = pytest.mark.gpu


def test_polygonize_spheres_golden(gpu):
    from paper_1903_11785_b200.mesh import polygonize
    from paper_1903_11785_b200.voxels import VoxelGrid

    z = G.load("spheres")
    rig, sils = G.rig(z), G.sils(z)
    sp = G.spec(z["carve3_spec"])
    grid = VoxelGrid(sp, G.unpack(z["carve3_occ"], sp.num_voxels))
    for mode, iso in (("exact", 0.5), ("fixed", 0.25)):
        m, st = polygonize(grid, rig, sils, mode=mode, fixed_isovalue=iso, object_id=4)
        assert np.array_equal(m.vertices, z[f"poly_{mode}_verts"]), mode
        assert np.array_equal(m.triangles, z[f"poly_{mode}_tris"]), mode
        assert np.all(m.object_ids == 4)
        assert [st.fallback_edges, st.inconsistent_starts] == list(z[f"poly_{mode}_stats"])


def test_single_voxel_kats(gpu):
    """tests/test_mesh.py:160-184, 239-245."""
    from paper_1903_11785_b200.mesh import polygonize
    from paper_1903_11785_b200.voxels import GridSpec, VoxelGrid

    z = G.load("spheres")
    rig = G.rig(z)
    spec = GridSpec(origin=(0, 0, 0), spacing=10.0, dims=(3, 3, 3))
    occ = np.zeros(27, dtype=bool)
    occ[spec.linear_index(1, 1, 1)] = True
    grid = VoxelGrid(spec, occ)
    allfg = [np.ones((c.image_height, c.image_width), dtype=bool) for c in rig]
    m, _ = polygonize(grid, rig, allfg, mode="exact")
    assert np.array_equal(m.vertices, z["single_exact_verts"])
    assert np.array_equal(m.triangles, z["single_exact_tris"])
    m, st = polygonize(grid, mode="fixed", fixed_isovalue=0.25)
    assert np.array_equal(m.vertices, z["single_fixed_verts"])
    assert np.array_equal(m.triangles, z["single_fixed_tris"])
    m, st = polygonize(grid, mode="fixed")
    assert m.num_triangles == 8 and len(m.vertices) == 6 and st.fallback_edges == 0
    for occ in (np.zeros(27, dtype=bool), np.ones(27, dtype=bool)):
        assert polygonize(VoxelGrid(spec, occ), mode="fixed")[0].num_triangles == 0
    with pytest.raises(ValueError):
        polygonize(grid, mode="exact")
    with pytest.raises(ValueError):
        polygonize(grid, mode="nope")


def test_polygonize_distorted_golden(gpu):
    from paper_1903_11785_b200.mesh import polygonize
    from paper_1903_11785_b200.voxels import VoxelGrid

    z = G.load("distorted")
    rig, sils = G.rig(z), G.sils(z)
    sp = G.spec(z["carve_spec"])
    grid = VoxelGrid(sp, G.unpack(z["carve_occ"], sp.num_voxels))
    m, st = polygonize(grid, rig, sils, mode="exact", object_id=2)
    assert np.array_equal(m.vertices, z["poly_verts"])
    assert np.array_equal(m.triangles, z["poly_tris"])
    assert [st.fallback_edges, st.inconsistent_starts] == list(z["poly_stats"])


@pytest.mark.parametrize("seed", range(4))
def test_polygonize_random_grids_vs_oracle(gpu, seed):
    """Random occupancies (dims incl. 1 and 2, ragged k words), both modes,
    batched in one launch."""
    from paper_1903_11785_b200.mesh import polygonize_grids
    from paper_1903_11785_b200.voxels import GridSpec, VoxelGrid

    z = G.load("spheres")
    rig, sils = G.rig(z), G.sils(z)
    rng = np.random.default_rng(seed)
    grids = []
    for _ in range(7):
        dims = tuple(int(d) for d in rng.integers(1, 40, 3))
        if rng.random() < 0.3:
            dims = (dims[0], dims[1], int(rng.choice([31, 32, 33, 64, 65])))
        spec = GridSpec(origin=rng.uniform(-600, -200, 3), spacing=float(rng.uniform(8, 40)),
                        dims=dims)
        occ = rng.random(spec.num_voxels) < rng.uniform(0.05, 0.9)
        grids.append(VoxelGrid(spec, occ))
    for mode in ("exact", "fixed"):
        batch = polygonize_grids(grids, rig, sils, mode, 0.3, object_ids=list(range(7)))
        for g, grid in enumerate(grids):
            sp = grid.spec
            v, t, o, st = O.polygonize(grid.occ, sp.origin, sp.spacing, sp.dims, rig, sils, mode,
                                       0.3, g)
            m = batch.mesh(g)
            assert np.array_equal(m.vertices, v), (mode, g, sp.dims)
            assert np.array_equal(m.triangles, t), (mode, g, sp.dims)
            assert np.array_equal(m.object_ids, o)
            s = batch.stats(g)
            assert [s.fallback_edges, s.inconsistent_starts] == \
                [st["fallback_edges"], st["inconsistent_starts"]]


def test_frame_roi_meshes_golden(gpu):
    """Per-ROI exact meshes of full frames (pipeline.py:175-190)."""
    from paper_1903_11785_b200.hull import Roi, dense_carve
    from paper_1903_11785_b200.mesh import TriangleMesh, polygonize_grids

    for name in ("tiny_cli", "figures"):
        z = G.load(name)
        rig, sils = G.rig(z), G.sils(z)
        rois = [Roi(r[:3], r[3:6], int(r[6])) for r in z["rois"]]
        grids = dense_carve(rig, sils, rois, float(z["fine_specs"][0][3]))
        batch = polygonize_grids(grids, rig, sils, "exact", 0.5,
                                 object_ids=[r.component_id for r in rois])
        for i in range(len(rois)):
            m = batch.mesh(i)
            assert np.array_equal(m.vertices, z[f"mesh{i}_verts"]), (name, i)
            assert np.array_equal(m.triangles, z[f"mesh{i}_tris"]), (name, i)
            assert np.array_equal(m.object_ids, z[f"mesh{i}_oids"]), (name, i)
        merged = batch.merged()
        assert np.array_equal(merged.vertices, z["merged_verts"])
        assert np.array_equal(merged.triangles, z["merged_tris"])
        ref = TriangleMesh.concatenate(batch.meshes())
        assert merged.num_triangles == ref.num_triangles


class TestEdgeIsovalue:
    """tests/test_mesh.py:63-140 known answers, through fvv_edge_isovalues."""

    @staticmethod
    def cam(i=0):
        from paper_1903_11785_b200.camera import CameraModel

        return CameraModel(id=i, image_width=200, image_height=100, fx=100.0, fy=100.0, cx=99.5,
                           cy=49.5)

    @staticmethod
    def half_plane(first_bg_u):
        s = np.zeros((100, 200), dtype=bool)
        s[:, :first_bg_u] = True
        return s

    def test_known_fractions(self, gpu):
        from paper_1903_11785_b200.mesh import edge_isovalue_cam

        cam = self.cam()
        z = 1000.0
        p_on = np.array([(50 - cam.cx) * z / cam.fx, 0.0, z])
        p_off = np.array([(150 - cam.cx) * z / cam.fx, 0.0, z])
        for boundary, expect in [(90, 0.4), (75, 0.25), (140, 0.9)]:
            lam, start_bg = edge_isovalue_cam(cam, self.half_plane(boundary), p_on, p_off)
            assert not start_bg and lam == pytest.approx(expect, abs=0.015)
        lam, start_bg = edge_isovalue_cam(cam, np.ones((100, 200), bool), [0, 0, 1000.0],
                                          [100, 0, 1000.0])
        assert lam == 1.0 and not start_bg
        lam, start_bg = edge_isovalue_cam(cam, np.zeros((100, 200), bool), [0, 0, 1000.0],
                                          [100, 0, 1000.0])
        assert lam == 0.0 and start_bg

    def test_min_over_cameras_ties_and_fallback(self, gpu):
        from paper_1903_11785_b200.camera import CameraRig
        from paper_1903_11785_b200.mesh import edge_isovalue

        rig = CameraRig([self.cam(i) for i in range(3)])
        z = 1000.0
        p_on = np.array([(50 - 99.5) * z / 100.0, 0.0, z])
        p_off = np.array([(150 - 99.5) * z / 100.0, 0.0, z])
        hit = edge_isovalue(rig, [self.half_plane(b) for b in (120, 90, 140)], p_on, p_off)
        assert hit.contributing_camera == 1
        hit = edge_isovalue(rig, [self.half_plane(90)] * 3, p_on, p_off)
        assert hit.contributing_camera == 0
        hit = edge_isovalue(rig, [np.ones((100, 200), bool)] * 3, [0, 0, -500.0],
                            [100, 0, -500.0])
        assert hit.lam == 0.5 and hit.contributing_camera == -1
