"""CPU checks of the C ABI boundary: libfvv.so loads without a GPU and
exports every entry point include/fvv.h declares; the Python binding's
record layouts match the header's structs."""

import ctypes
import os
import re

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared():
    src = open(os.path.join(ROOT, "include", "fvv.h")).read()
    return sorted(set(re.findall(r"\b(fvv_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_1903_11785_b200 import _lib

    lib = ctypes.CDLL(_lib.LIB_PATH)
    names = declared()
    assert names, "no entry points found in include/fvv.h"
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    assert set(_lib.SYMBOLS) <= set(names)
    assert lib.fvv_version() >= 1


def test_record_layouts_match_header():
    from paper_1903_11785_b200 import _lib

    import oracle

    assert _lib.CAM_DTYPE.itemsize == 192 and oracle.CAM_DTYPE == _lib.CAM_DTYPE
    assert _lib.GRID_DTYPE.itemsize == 56
    assert _lib.COMP_DTYPE.itemsize == 64
    # every record the binding builds has the size the compiled library uses
    sizes = np.zeros(8, dtype=np.int64)
    assert _lib.load().fvv_abi_sizes(_lib.host_ptr(sizes), 8) == 8
    assert list(sizes) == [_lib.CAM_DTYPE.itemsize, _lib.GRID_DTYPE.itemsize,
                           _lib.COMP_DTYPE.itemsize, _lib.FRAME_CONFIG_DTYPE.itemsize,
                           _lib.FRAME_STATS_DTYPE.itemsize, ctypes.sizeof(_lib.FrameOutputs),
                           ctypes.sizeof(_lib.SeqConfig), ctypes.sizeof(_lib.SeqResultInfo)]


def test_hot_path_refuses_to_run_without_cuda():
    import pytest
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_1903_11785_b200 import hull
    from paper_1903_11785_b200.camera import CameraModel, CameraRig
    from paper_1903_11785_b200.voxels import GridSpec

    rig = CameraRig([CameraModel(id=0, image_width=4, image_height=4, fx=1.0, fy=1.0, cx=1.5,
                                 cy=1.5)])
    with pytest.raises(RuntimeError, match="CUDA"):
        hull.carve(rig, [np.ones((4, 4), bool)], GridSpec((0, 0, 0), 1.0, (2, 2, 2)))
