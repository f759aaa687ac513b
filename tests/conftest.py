import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def _ensure_built():
    """Build libplora.so and the oracle checkers when missing (no-op on the GPU
    box, where the prebuilt .so files travel with the snapshot)."""
    lib = os.path.join(ROOT, "paper_2512_20210_b200", "libplora.so")
    if not os.path.exists(lib):
        subprocess.run(["make", "-C", os.path.join(ROOT, "paper_2512_20210_b200", "csrc"),
                        "-j8"], check=True)
    if not os.path.exists(os.path.join(ROOT, "oracle", "liboracle.so")):
        subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "all"], check=True)
    ref = os.path.join(ROOT, "oracle", "_ref", "libref.so")
    if not os.path.exists(ref) and os.path.isdir("/root/reference/proj"):
        subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "ref"], check=True)


_ensure_built()


@pytest.fixture(scope="session")
def ref():
    from oracle import ref as R
    if not R.available():
        pytest.skip("oracle/_ref/libref.so (reference build) not present")
    return R


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda:0")
