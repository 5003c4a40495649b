"""B200-native free-viewpoint-video synthesis (drop-in for the reference
``freeview`` package's hot path: carve -> CCL/ROI -> ROI carve -> exact
marching cubes -> visibility -> view-dependent colour).

Host code mirrors the reference's modules (camera, voxels, hull, mesh,
visibility, render, pipeline); every stage computes in hand-written sm_100a
CUDA kernels behind the C ABI in include/fvv.h (libfvv.so).
"""

from .camera import CalibrationError, CameraModel, CameraRig, load_rig, project
from .voxels import GridSpec, VoxelGrid

__all__ = [
    "CalibrationError",
    "CameraModel",
    "CameraRig",
    "load_rig",
    "project",
    "GridSpec",
    "VoxelGrid",
]

__version__ = "0.1.0"
