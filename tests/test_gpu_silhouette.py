"""GPU parity for silhouette extraction (silhouette.py) and
run_frame's proposal path against the reference's golden outputs."""

import json

import numpy as np
import pytest

import golden_io as G
import oracle as O

pytestmark = pytest.mark.gpu


def test_distance_map_background_extraction_golden(gpu):
    from paper_1903_11785_b200.silhouette import (AdaptiveParams, build_background,
                                                   distance_map, extract_silhouette)

    z = G.load("silhouette")
    rig = G.rig(z)
    cfg = json.loads(str(z["cfg"]))
    params = AdaptiveParams(cfg["theta_near"], cfg["theta_far"], cfg["d_max"])
    for i, c in enumerate(rig):
        h, w = c.image_height, c.image_width
        prop = G.unpack(z[f"prop{i}"], h * w).reshape(h, w)
        dm = distance_map(prop)
        assert np.array_equal(dm, z[f"dm{i}"]), i
        bg = build_background(list(z[f"bgframes{i}"]))
        if i < 2:
            assert np.array_equal(bg.mean, z[f"bgmean{i}"])
            assert np.array_equal(bg.std, z[f"bgstd{i}"])
        sil = extract_silhouette(z[f"frame{i}"], bg, dm, params)
        assert np.array_equal(sil, G.unpack(z[f"sil{i}"], h * w).reshape(h, w)), i
    assert np.all(np.isinf(distance_map(np.zeros((5, 7), bool))))
    one = np.zeros((40, 50), dtype=bool)
    one[3, 47] = True
    assert np.array_equal(distance_map(one), z["dm_one"])
    rnd = G.unpack(z["rnd_prop"], 61 * 83).reshape(61, 83)
    assert np.array_equal(distance_map(rnd), z["dm_rnd"])
    with pytest.raises(ValueError):
        distance_map(np.zeros((4, 4, 3), bool))
    with pytest.raises(ValueError):
        build_background([z["frame0"]])


@pytest.mark.parametrize("shape,density", [((1080, 1920), 0.002), ((300, 517), 0.05),
                                           ((64, 4000), 0.01), ((2000, 33), 0.2)])
def test_distance_map_vs_oracle(gpu, shape, density):
    from paper_1903_11785_b200.silhouette import distance_map

    rng = np.random.default_rng(int(density * 1000))
    prop = rng.random(shape) < density
    assert np.array_equal(distance_map(prop), O.distance_map(prop))


def test_run_frame_proposal_path_golden(gpu):
    """run_frame(sils=None, proposals, background) (pipeline.py:126-137)."""
    from paper_1903_11785_b200.pipeline import PipelineConfig, run_frame
    from paper_1903_11785_b200.silhouette import build_background

    z = G.load("silhouette")
    rig = G.rig(z)
    d = json.loads(str(z["cfg"]))
    d["t_large"] = float("inf")
    cfg = PipelineConfig(**{k: (tuple(v) if isinstance(v, list) else v) for k, v in d.items()})
    frames = {c.id: z[f"frame{i}"] for i, c in enumerate(rig)}
    proposals = {c.id: G.unpack(z[f"prop{i}"], c.image_height * c.image_width)
                 .reshape(c.image_height, c.image_width) for i, c in enumerate(rig)}
    background = {c.id: build_background(list(z[f"bgframes{i}"])) for i, c in enumerate(rig)}
    bundle = run_frame(cfg, rig, frames, proposals=proposals, background=background)
    assert bundle.stats == json.loads(str(z["stats"]))
