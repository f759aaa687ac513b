"""The C++ face (include/plora.hpp) compiles against the C ABI and behaves
like lorasim::PagePool (reference tests re-expressed in C++)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_cpp_dropin(tmp_path):
    exe = tmp_path / "dropin"
    lib_dir = os.path.join(ROOT, "paper_2512_20210_b200")
    subprocess.run(["g++", "-std=c++17", "-O1", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "dropin_pagepool.cpp"), "-L", lib_dir,
                    "-lplora", f"-Wl,-rpath,{lib_dir}", "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True)
    assert out.returncode == 0, out.stderr
    assert "dropin ok" in out.stdout


def _build_device_dropin(tmp_path):
    exe = tmp_path / "dropin_device"
    lib_dir = os.path.join(ROOT, "paper_2512_20210_b200")
    subprocess.run(["g++", "-std=c++17", "-O1", "-I", os.path.join(ROOT, "include"),
                    "-I", "/usr/local/cuda/include",
                    os.path.join(ROOT, "tests", "cpp", "dropin_device.cpp"), "-L", lib_dir,
                    "-lplora", f"-Wl,-rpath,{lib_dir}", "-L", "/usr/local/cuda/lib64", "-lcudart",
                    "-Wl,-rpath,/usr/local/cuda/lib64", "-o", str(exe)], check=True)
    return exe


def test_cpp_dropin_device_builds(tmp_path):
    """The device half of the C++ face (DeviceStore, BatchPlan, bgmv,
    sgmv_layer, sgmv_fused) compiles and links against the C ABI."""
    assert _build_device_dropin(tmp_path).exists()


@pytest.mark.gpu
def test_cpp_dropin_device_runs(tmp_path, cuda):
    """A C++ caller drives pool -> store -> plan -> bgmv / sgmv_layer and
    matches a double-precision host computation."""
    out = subprocess.run([str(_build_device_dropin(tmp_path))], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "dropin device ok" in out.stdout
