"""The reference's Sphere/Box scene generator on the GPU (SURVEY.md 8f4,
synthetic.py:165-243) against outputs of the reference itself
(tests/golden/synth.npz, scripts/make_golden.py): silhouettes, noiseless
and noisy frames, eroded proposals, bit for bit."""

import numpy as np
import pytest

import golden_io as G

pytestmark = pytest.mark.gpu


def _scene():
    from paper_1903_11785_b200 import synthetic as S

    objs = [S.Sphere(center=[-350, 0, 450], radius=250),
            S.Box(lo=[300, -200, 200], hi=[700, 200, 700], color=[70, 110, 200]),
            S.Sphere(center=[0, 400, 300], radius=120, color=[90, 200, 120])]
    z = G.load("synth")
    rig = G.rig(z)
    return z, rig, objs, S.SyntheticScene(rig=rig, objects=objs)


def test_silhouettes_and_proposals_match_reference(gpu):
    from paper_1903_11785_b200 import synthetic as S

    z, rig, objs, scene = _scene()
    sils = S.scene_silhouettes(scene)
    for i, cam in enumerate(rig):
        h, w = cam.image_height, cam.image_width
        assert np.array_equal(sils[i], G.unpack(z[f"sil{i}"], h * w).reshape(h, w)), i
        assert sils[i].any() and not sils[i].all()
        assert np.array_equal(S.proposal_from_silhouette(sils[i], 3),
                              G.unpack(z[f"prop{i}"], h * w).reshape(h, w)), i
        assert np.array_equal(S.proposal_from_silhouette(sils[i], 1),
                              G.unpack(z[f"prop1_{i}"], h * w).reshape(h, w)), i


def test_frames_match_reference(gpu):
    from paper_1903_11785_b200 import synthetic as S

    z, rig, objs, scene = _scene()
    for i, cam in enumerate(rig):
        assert np.array_equal(S.shade_frame(scene, cam, 0.0, 0), z[f"frame{i}"]), i
        assert np.array_equal(S.shade_frame(scene, cam, 1.5, 3), z[f"noisy{i}"]), i
    frames = S.scene_frames(scene)
    assert np.array_equal(frames[0], z["frame0"])


def test_scene_api_errors(gpu):
    from paper_1903_11785_b200 import synthetic as S

    with pytest.raises(ValueError, match="radius"):
        S.Sphere(center=[0, 0, 0], radius=0)
    with pytest.raises(ValueError, match="positive extent"):
        S.Box(lo=[0, 0, 0], hi=[0, 1, 1])
    with pytest.raises(ValueError, match="outside the stage"):
        S.validate_in_stage([S.Sphere(center=[0, 0, 0], radius=10)], [-5, -5, -5], [5, 5, 5])
