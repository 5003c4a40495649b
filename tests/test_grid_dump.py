"""RLE grid dump (voxels.py:100-162 save_grid / load_grid, formats.md):
files byte-identical to the ones the reference wrote (tests/golden/
grid_dump.npz, scripts/make_golden.py)."""

import struct

import numpy as np
import pytest

import golden_io as G
import oracle as O

HEAD = "<4sI3Iq d 3d"


def _cases():
    z = G.load("grid_dump")
    i = 0
    while f"g{i}_dims" in z.files:
        dims = tuple(int(d) for d in z[f"g{i}_dims"])
        n = int(np.prod(dims))
        yield (i, dims, z[f"g{i}_origin"], float(z[f"g{i}_spacing"]),
               G.unpack(z[f"g{i}_occ"], n), z[f"g{i}_file"].tobytes())
        i += 1


def test_oracle_runs_match_reference_files():
    for i, dims, origin, spacing, occ, raw in _cases():
        nruns = struct.unpack(HEAD, raw[:struct.calcsize(HEAD)])[5]
        runs = np.frombuffer(raw[struct.calcsize(HEAD):], dtype="<u8", count=nruns)
        assert np.array_equal(O.rle_runs(occ), runs), i


def test_load_grid_reads_reference_files(tmp_path):
    from paper_1903_11785_b200.voxels import load_grid

    for i, dims, origin, spacing, occ, raw in _cases():
        path = tmp_path / f"g{i}.bin"
        path.write_bytes(raw)
        g = load_grid(path)
        assert g.spec.dims == dims and g.spec.spacing == spacing
        assert np.array_equal(g.spec.origin, origin)
        assert np.array_equal(g.occ, occ), i


def test_load_grid_errors(tmp_path):
    from paper_1903_11785_b200.voxels import load_grid

    bad = tmp_path / "not_a_grid.bin"
    bad.write_bytes(b"XXXX" + b"\0" * 100)
    with pytest.raises(ValueError, match="not a voxel grid"):
        load_grid(bad)
    head = struct.pack(HEAD, b"FVVG", 2, 1, 1, 1, 0, 1.0, 0.0, 0.0, 0.0)
    ver = tmp_path / "v2.bin"
    ver.write_bytes(head)
    with pytest.raises(ValueError, match="unsupported grid dump version"):
        load_grid(ver)
    short = tmp_path / "short.bin"
    short.write_bytes(struct.pack(HEAD, b"FVVG", 1, 2, 2, 1, 1, 1.0, 0.0, 0.0, 0.0) +
                      np.array([3], dtype="<u8").tobytes())
    with pytest.raises(ValueError, match="do not cover"):
        load_grid(short)


@pytest.mark.gpu
def test_save_grid_byte_identical(gpu, tmp_path):
    """save_grid (bit transitions found on the GPU) writes the reference's
    bytes, from a host array and from a carved device bit field."""
    from paper_1903_11785_b200.voxels import GridSpec, VoxelGrid, save_grid

    for i, dims, origin, spacing, occ, raw in _cases():
        spec = GridSpec(origin=origin, spacing=spacing, dims=dims)
        path = tmp_path / f"g{i}.bin"
        save_grid(VoxelGrid(spec=spec, occ=occ), path)
        assert path.read_bytes() == raw, i
        dev = VoxelGrid(spec=spec, occ=occ)
        dev._bits = dev.device_bits()
        dev._occ = None  # force the device path
        save_grid(dev, path)
        assert path.read_bytes() == raw, i


@pytest.mark.gpu
def test_save_load_random_patterns(gpu, tmp_path):
    from paper_1903_11785_b200.voxels import GridSpec, VoxelGrid, load_grid, save_grid

    rng = np.random.default_rng(5)
    for n in (1, 2, 31, 32, 33, 63, 64, 65, 1000, 4097):
        for p in (0.0, 0.2, 0.5, 1.0):
            occ = rng.random(n) < p
            spec = GridSpec(origin=(0, 0, 0), spacing=1.0, dims=(n, 1, 1))
            path = tmp_path / "g.bin"
            save_grid(VoxelGrid(spec=spec, occ=occ), path)
            assert np.array_equal(load_grid(path).occ, occ)
            runs = np.frombuffer(path.read_bytes()[struct.calcsize(HEAD):], dtype="<u8")
            assert np.array_equal(runs, O.rle_runs(occ))
