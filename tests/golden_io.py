"""Load tests/golden/*.npz fixtures (written by scripts/make_golden.py from
the reference itself) into this repo's host types."""

from __future__ import annotations

import json
import os

import numpy as np

from paper_1903_11785_b200.camera import CameraModel, CameraRig
from paper_1903_11785_b200.voxels import GridSpec

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    return np.load(os.path.join(GOLDEN, name + ".npz"))


def rig(z, key="rig"):
    return CameraRig([CameraModel.from_dict(d) for d in json.loads(str(z[key]))["cameras"]])


def camera(z, key):
    return CameraModel.from_dict(json.loads(str(z[key])))


def unpack(bits, n):
    return np.unpackbits(np.asarray(bits, dtype=np.uint8), bitorder="little")[:n].astype(bool)


def sils(z):
    shapes = z["sil_shapes"]
    if "sils" in z.files:
        return [unpack(z["sils"][i], int(h * w)).reshape(h, w) for i, (h, w) in enumerate(shapes)]
    out, off = [], 0
    flat = z["sil_list"]
    for h, w in shapes:
        nbytes = (int(h * w) + 7) // 8
        out.append(unpack(flat[off:off + nbytes], int(h * w)).reshape(h, w))
        off += nbytes
    return out


def spec(arr):
    arr = np.asarray(arr, dtype=np.float64)
    return GridSpec(origin=arr[:3], spacing=float(arr[3]), dims=tuple(int(d) for d in arr[4:7]))


def frames(z, r):
    return {c.id: z["frames"][i] for i, c in enumerate(r)}
