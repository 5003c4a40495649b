import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))


def pytest_sessionstart(session):
    """Build libfvv.so when a checkout has none yet (nvcc cross-compiles
    without a GPU); a GPU box receives the prebuilt library."""
    import shutil
    import subprocess

    lib = os.path.join(ROOT, "paper_1903_11785_b200", "libfvv.so")
    if not os.path.exists(lib) and shutil.which("make") and (
            shutil.which("nvcc") or os.path.exists("/usr/local/cuda/bin/nvcc")):
        subprocess.run(["make", "-s", "-j8", "-C",
                        os.path.join(ROOT, "paper_1903_11785_b200", "csrc")], check=False)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity tests proper")
    config.addinivalue_line("markers", "reference: imports the reference from /root/reference")


def has_gpu():
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False


@pytest.fixture(scope="session")
def gpu():
    if not has_gpu():
        pytest.skip("no CUDA device")
    import paper_1903_11785_b200._lib as L

    L.load()  # fail loudly if libfvv.so is missing on a GPU box
    return True
