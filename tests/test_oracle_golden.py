"""Pin the CPU oracle (oracle/) to the reference's own outputs.

Every fixture in tests/golden/ was produced by running the reference
implementation (scripts/make_golden.py); the oracle must reproduce each
one bit for bit. CPU only — these run in the driver's `-m "not gpu"` pass.
"""

import json

import numpy as np
import pytest

import golden_io as G
import oracle as O


def test_tiny_cli_matches_reference_manifest_stats():
    """TINY_SPEC golden: the reference's committed bundle manifest
    (pkg/frontend/tests/fixtures/bundle/manifest.json:29-38)."""
    z = G.load("tiny_cli")
    rig = G.rig(z)
    cfg = json.loads(str(z["cfg"]))
    out = O.run_frame(rig, G.sils(z), cfg["stage_lo"], cfg["stage_hi"], cfg["coarse_spacing"],
                      cfg["fine_spacing"], cfg["min_views"], cfg["t_small"], np.inf,
                      cfg["roi_margin"], cfg["t_v"], keep_depths=True)
    assert out["stats"] == json.loads(str(z["stats"]))
    assert out["stats"]["triangles"] == 3292 and out["stats"]["sparse_occupied"] == 315


@pytest.mark.parametrize("name", ["tiny_cli", "figures"])
def test_full_frame_matches_reference(name):
    z = G.load(name)
    rig = G.rig(z)
    sils = G.sils(z)
    cfg = json.loads(str(z["cfg"]))
    t_large = np.inf if cfg["t_large"] is None else cfg["t_large"]
    out = O.run_frame(rig, sils, cfg["stage_lo"], cfg["stage_hi"], cfg["coarse_spacing"],
                      cfg["fine_spacing"], cfg["min_views"], cfg["t_small"], t_large,
                      cfg["roi_margin"], cfg["t_v"], keep_depths=True)
    assert out["stats"] == json.loads(str(z["stats"]))
    origin, s, dims, occ = out["coarse"]
    assert np.array_equal(occ, G.unpack(z["coarse_occ"], len(occ)))
    assert np.array_equal(out["labels"], z["labels"])
    comps = np.array([[c.id, c.voxel_count, *c.bbox_min, *c.bbox_max] for c in out["components"]],
                     dtype=np.int64).reshape(-1, 8)
    assert np.array_equal(comps, z["comps"])
    assert [c.id for c in out["filtered_components"]] == list(z["fcomps"])
    rois = np.array([list(lo) + list(hi) + [cid] for lo, hi, cid in out["rois"]]).reshape(-1, 7)
    assert np.array_equal(rois, z["rois"])
    for i, (fo, fs, fd, focc) in enumerate(out["fine"]):
        assert np.array_equal(np.array(list(fo) + [fs] + list(fd)), z["fine_specs"][i])
        assert np.array_equal(focc, G.unpack(z[f"fine{i}_occ"], len(focc)))
    for i, (v, t, o) in enumerate(out["meshes"]):
        assert np.array_equal(v, z[f"mesh{i}_verts"])
        assert np.array_equal(t, z[f"mesh{i}_tris"])
        assert np.array_equal(o, z[f"mesh{i}_oids"])
    mv, mt, mo = out["merged"]
    assert np.array_equal(mv, z["merged_verts"]) and np.array_equal(mt, z["merged_tris"])
    for i, c in enumerate(rig):
        assert np.array_equal(out["visibility"][c.id], G.unpack(z["vis"][i], len(mt)))
    assert np.array_equal(out["depths"][rig[0].id], z["depth0"])
    # E: virtual view (render.py:64-113) and its raster
    virtual = G.camera(z, "virtual")
    depth, tid = O.rasterize(mv, mt, virtual)
    assert np.array_equal(depth, z["virtual_depth"]) and np.array_equal(tid, z["virtual_tri_id"])
    color, source, covered = O.render_view(mv, mt, rig, G.frames(z, rig), out["visibility"],
                                           virtual)
    assert np.array_equal(source, z["render_source"])
    assert np.array_equal(color, z["render_color"])


def test_spheres_carve_polygonize_visibility():
    z = G.load("spheres")
    rig = G.rig(z)
    sils = G.sils(z)
    for i in range(4):
        sp = G.spec(z[f"carve{i}_spec"])
        occ = O.carve(rig, sils, sp.origin, sp.spacing, sp.dims, int(z[f"carve{i}_minv"]))
        assert np.array_equal(occ, G.unpack(z[f"carve{i}_occ"], sp.num_voxels)), i
    sp = G.spec(z["carve3_spec"])
    occ = G.unpack(z["carve3_occ"], sp.num_voxels)
    for mode, iso in (("exact", 0.5), ("fixed", 0.25)):
        v, t, o, st = O.polygonize(occ, sp.origin, sp.spacing, sp.dims, rig, sils, mode, iso, 4)
        assert np.array_equal(v, z[f"poly_{mode}_verts"])
        assert np.array_equal(t, z[f"poly_{mode}_tris"])
        assert [st["fallback_edges"], st["inconsistent_starts"]] == list(z[f"poly_{mode}_stats"])
    # single-voxel KATs
    sv = (np.zeros(3), 10.0, (3, 3, 3))
    socc = np.zeros(27, dtype=bool)
    socc[13] = True
    allfg = [np.ones((c.image_height, c.image_width), dtype=bool) for c in rig]
    v, t, _, _ = O.polygonize(socc, *sv, rig, allfg, "exact")
    assert np.array_equal(v, z["single_exact_verts"]) and np.array_equal(t, z["single_exact_tris"])
    v, t, _, _ = O.polygonize(socc, *sv, mode="fixed", fixed_isovalue=0.25)
    assert np.array_equal(v, z["single_fixed_verts"]) and np.array_equal(t, z["single_fixed_tris"])
    # visibility maps over every camera
    verts, tris = z["vis_verts"], z["vis_tris"]
    for i, c in enumerate(rig):
        depth, _ = O.rasterize(verts, tris, c)
        if i == 0:
            assert np.array_equal(depth, z["vis_depth0"])
        assert np.array_equal(O.classify(verts, tris, c, depth, 150.0),
                              G.unpack(z["vis_flags"][i], len(tris)))
    depth, tid = O.rasterize(verts, tris, rig[5])
    assert np.array_equal(depth, z["raster5_depth"]) and np.array_equal(tid, z["raster5_tri_id"])


def test_distorted_cameras_project_carve_isovalues():
    z = G.load("distorted")
    rig = G.rig(z)
    sils = G.sils(z)
    pts = z["pts"]
    for ci, c in enumerate(rig):
        px, zz, inside = O.project(c, pts)
        assert np.array_equal(px, z[f"proj{ci}_px"])
        assert np.array_equal(zz, z[f"proj{ci}_z"])
        assert np.array_equal(inside, z[f"proj{ci}_in"])
        px1, z1, in1 = O.project(c, pts[ci:ci + 1])  # one point: numpy's gemv order
        assert np.array_equal(np.array([px1[0, 0], px1[0, 1], z1[0], float(in1[0])]),
                              z[f"proj{ci}_single"])
        px, _, _ = O.project(c, pts, use_distortion=False)
        assert np.array_equal(px, z[f"projnd{ci}_px"])
    sp = G.spec(z["carve_spec"])
    occ = O.carve(rig, sils, sp.origin, sp.spacing, sp.dims)
    assert np.array_equal(occ, G.unpack(z["carve_occ"], sp.num_voxels))
    v, t, _, st = O.polygonize(occ, sp.origin, sp.spacing, sp.dims, rig, sils, "exact", 0.5, 2)
    assert np.array_equal(v, z["poly_verts"]) and np.array_equal(t, z["poly_tris"])
    assert [st["fallback_edges"], st["inconsistent_starts"]] == list(z["poly_stats"])


def test_ccl_random_grids():
    z = G.load("ccl")
    i = 0
    while f"g{i}_dims" in z.files:
        dims = tuple(int(d) for d in z[f"g{i}_dims"])
        n = dims[0] * dims[1] * dims[2]
        occ = G.unpack(z[f"g{i}_occ"], n)
        labels, comps = O.label(occ, dims)
        assert np.array_equal(labels, z[f"g{i}_labels"]), i
        arr = np.array([[c.id, c.voxel_count, *c.bbox_min, *c.bbox_max] for c in comps],
                       dtype=np.int64).reshape(-1, 8)
        assert np.array_equal(arr, z[f"g{i}_comps"]), i
        _, flabels, _ = O.filter_noise(labels, comps, 3, 40)
        assert np.array_equal(flabels, z[f"g{i}_flabels"]), i
        i += 1
    assert i == 8


def test_raster_ties_winding_and_visibility():
    z = G.load("raster")
    cam = G.camera(z, "cam")
    depth, tid = O.rasterize(z["verts"], z["tris"], cam)
    assert np.array_equal(depth, z["depth"])
    assert np.array_equal(tid, z["tri_id"])
    assert np.array_equal(O.classify(z["verts"], z["tris"], cam, depth, 50.0), z["vis"])
    one = z["one_verts"]
    d1, _ = O.rasterize(one, [[0, 1, 2]], cam)
    assert np.array_equal(O.classify(one, [[0, 1, 2]], cam, d1, 10.0), z["one_vis"])


def test_silhouette_extraction_matches_reference():
    """silhouette.py: exact EDT, background statistics, adaptive threshold."""
    z = G.load("silhouette")
    rig = G.rig(z)
    cfg = json.loads(str(z["cfg"]))
    for i, c in enumerate(rig):
        h, w = c.image_height, c.image_width
        prop = G.unpack(z[f"prop{i}"], h * w).reshape(h, w)
        dm = O.distance_map(prop)
        assert np.array_equal(dm, z[f"dm{i}"]), i
        mean, std = O.build_background(list(z[f"bgframes{i}"]))
        if i < 2:
            assert np.array_equal(mean, z[f"bgmean{i}"]) and np.array_equal(std, z[f"bgstd{i}"])
        sil = O.extract_silhouette(z[f"frame{i}"], mean, std, dm, cfg["theta_near"],
                                   cfg["theta_far"], cfg["d_max"])
        assert np.array_equal(sil, G.unpack(z[f"sil{i}"], h * w).reshape(h, w)), i
    assert np.all(np.isinf(O.distance_map(np.zeros((5, 7), bool))))
    one = np.zeros((40, 50), dtype=bool)
    one[3, 47] = True
    assert np.array_equal(O.distance_map(one), z["dm_one"])
    rnd = G.unpack(z["rnd_prop"], 61 * 83).reshape(61, 83)
    assert np.array_equal(O.distance_map(rnd), z["dm_rnd"])
