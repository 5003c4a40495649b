"""f3: the bundle writer produces the reference's exact bytes
(tests/golden/bundle_sha256.json was written by the reference's own
write_bundle, scripts/make_golden.py fixture_bundle). CPU: the bundle is
assembled from the reference's golden arrays and the oracle's depth planes;
GPU: straight from run_frame."""

import hashlib
import json
import os

import numpy as np
import pytest

import golden_io as G
import oracle as O

GOLD = json.load(open(os.path.join(G.GOLDEN, "bundle_sha256.json")))


def _hashes(root):
    out = {}
    for d, _, files in os.walk(root):
        for fn in files:
            rel = os.path.relpath(os.path.join(d, fn), root)
            if rel != "timings.json":
                out[rel] = hashlib.sha256(open(os.path.join(d, fn), "rb").read()).hexdigest()
    return dict(sorted(out.items()))


def _cfg(z):
    from paper_1903_11785_b200.pipeline import PipelineConfig

    d = json.loads(str(z["cfg"]))
    d["t_large"] = float("inf") if d["t_large"] is None else d["t_large"]
    return PipelineConfig(**{k: (tuple(v) if isinstance(v, list) else v) for k, v in d.items()})


def test_bundle_bytes_match_reference_cpu(tmp_path):
    from paper_1903_11785_b200.bundle import SceneBundle, load_bundle, write_bundle
    from paper_1903_11785_b200.mesh import TriangleMesh

    z = G.load("tiny_cli")
    rig = G.rig(z)
    cfg = _cfg(z)
    meshes, i = [], 0
    while f"mesh{i}_verts" in z.files:
        meshes.append(TriangleMesh(z[f"mesh{i}_verts"], z[f"mesh{i}_tris"], z[f"mesh{i}_oids"]))
        i += 1
    merged = TriangleMesh.concatenate(meshes)
    vis = {c.id: G.unpack(z["vis"][k], merged.num_triangles) for k, c in enumerate(rig)}
    depths = {c.id: O.rasterize(merged.vertices, merged.triangles, c)[0] for c in rig}
    b = SceneBundle(frame_id=7, rig=rig, meshes=meshes, textures=G.frames(z, rig),
                    visibility=vis, stats=json.loads(str(z["stats"])),
                    stage_lo=np.array(cfg.stage_lo), stage_hi=np.array(cfg.stage_hi),
                    depths=depths)
    write_bundle(b, tmp_path, export_depth=True)
    assert _hashes(tmp_path) == GOLD
    back = load_bundle(tmp_path)
    assert back.stats == b.stats and back.frame_id == 7
    assert np.array_equal(back.merged_mesh.triangles, merged.triangles)
    assert all(np.array_equal(back.visibility[c.id], vis[c.id]) for c in rig)


@pytest.mark.gpu
def test_bundle_bytes_match_reference_gpu(gpu, tmp_path):
    from paper_1903_11785_b200.bundle import BundleWriter
    from paper_1903_11785_b200.pipeline import run_frame

    z = G.load("tiny_cli")
    rig = G.rig(z)
    bundle = run_frame(_cfg(z), rig, G.frames(z, rig), sils=G.sils(z), frame_id=7,
                       keep_depths=True)
    with BundleWriter() as w:
        w.submit(bundle, tmp_path, export_depth=True)
    assert _hashes(tmp_path) == GOLD
