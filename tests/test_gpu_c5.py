"""C5 kernel-sweep parity (BASELINE.json configs[4]): B-1 carve
and B-2 26-connected CCL of a TRUE n^3 stage grid, n in {512, 1024}, for ring
rigs of 4, 16 and 64 1080p cameras, bit for bit against the CPU oracle.

The reference caps grids at 400 M voxels (voxels.py:15); 1024^3 = 1.07 G
voxels lifts that budget explicitly on both sides (GridSpec(budget=...) here,
the oracle takes dims as given). This is where the certified-FP32 carve is
stressed hardest: the widest Z ranges per tile, the largest pixel rectangles
per 16^3 tile (64 cameras see the cube from every side) and the float64
queue. Occupancy is compared as packed bits, labels chunk by chunk, so the
1024^3 cases stay within a few GB of host memory."""

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu

SIDE = 8000.0  # mm: cube stage (-4000, -4000, 0) .. (4000, 4000, 8000)


def _scene(ncam):
    from paper_1903_11785_b200 import synthetic as S

    rig = S.ring_rig(ncam, (0, 0, 1000), 15000, 4000, 1920, 1080, 1600)
    objs = S.place_figures(12, (-3000, -3000), (3000, 3000), seed=0)  # C3 figures, in the cube
    masks, _ = S.render_scene_device(rig, objs, shade=False)
    return rig, masks


@pytest.mark.parametrize("n", [512, 1024])
@pytest.mark.parametrize("ncam", [4, 16, 64])
def test_c5_cube_carve_and_ccl_match_oracle(gpu, n, ncam):
    import torch

    from paper_1903_11785_b200.hull import carve, label_components
    from paper_1903_11785_b200.voxels import GridSpec

    rig, masks = _scene(ncam)
    spec = GridSpec(origin=(-SIDE / 2, -SIDE / 2, 0.0), spacing=SIDE / n, dims=(n, n, n),
                    budget=n ** 3)
    grid = carve(rig, masks, spec)
    m_np = [m.cpu().numpy().astype(bool) for m in masks]
    ref = O.carve(list(rig), m_np, spec.origin, spec.spacing, spec.dims)
    nvox = n ** 3
    got_bits = grid.device_bits().cpu().numpy().view(np.uint8)[:nvox // 8]
    assert np.array_equal(got_bits, np.packbits(ref, bitorder="little")), (n, ncam)
    assert grid.occupied_count == int(ref.sum()) > 0

    lab = label_components(grid)
    ref_labels, ref_comps = O.label(ref, spec.dims)
    del ref
    assert [(c.id, c.voxel_count, tuple(c.bbox_min), tuple(c.bbox_max))
            for c in lab.components] == \
        [(c.id, c.voxel_count, tuple(c.bbox_min), tuple(c.bbox_max)) for c in ref_comps]
    dev = lab.device_labels()
    step = 1 << 26
    for a in range(0, nvox, step):
        assert np.array_equal(dev[a:a + step].cpu().numpy(), ref_labels[a:a + step]), (n, ncam, a)
    del dev
    torch.cuda.empty_cache()


def test_c5_carve_is_independent_of_grid_batching(gpu):
    """Size-independent property at 1024^3: carving the cube as one grid or
    as its 8 octant sub-grids (one batched launch) sets the same voxels."""
    from paper_1903_11785_b200._device import DeviceSilhouettes
    from paper_1903_11785_b200.hull import carve_grids
    from paper_1903_11785_b200.voxels import GridSpec

    n, h = 1024, 512
    rig, masks = _scene(16)
    ds = DeviceSilhouettes(rig, masks)
    s = SIDE / n
    whole = GridSpec(origin=(-SIDE / 2, -SIDE / 2, 0.0), spacing=s, dims=(n, n, n), budget=n ** 3)
    octs = [GridSpec(origin=(-SIDE / 2 + i * h * s, -SIDE / 2 + j * h * s, k * h * s), spacing=s,
                     dims=(h, h, h)) for k in (0, 1) for j in (0, 1) for i in (0, 1)]
    big = carve_grids(ds, [whole])[0].occ.reshape(n, n, n)  # [k, j, i]
    parts = carve_grids(ds, octs)
    for g, (k, j, i) in zip(parts, [(k, j, i) for k in (0, 1) for j in (0, 1) for i in (0, 1)]):
        sub = big[k * h:(k + 1) * h, j * h:(j + 1) * h, i * h:(i + 1) * h]
        assert np.array_equal(g.occ.reshape(h, h, h), sub), (k, j, i)
