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


REF_INC = "/root/reference/proj/include"


def _nlohmann():
    import sys
    for d in sys.path:
        p = os.path.join(d, "include", "cudnn_frontend", "thirdparty")
        if d and os.path.isdir(os.path.join(p, "nlohmann")):
            return p
    return None


@pytest.mark.skipif(not os.path.isdir(REF_INC) or not os.path.exists(
    os.path.join(ROOT, "oracle", "_ref", "libref.so")), reason="needs the reference build")
def test_engine_excerpt_against_reference(tmp_path):
    """The reference engine's pool call sites (engine.cpp:77-78, 293, 299, 489,
    587) compile against lorasim's own types with libplora's pool
    (include/plora_lorasim.hpp) next to the reference BlockArena, and a churn
    through them matches the reference lorasim::PagePool step for step."""
    nl = _nlohmann()
    if nl is None:
        pytest.skip("nlohmann/json not found")
    exe = tmp_path / "engine_excerpt"
    lib_dir = os.path.join(ROOT, "paper_2512_20210_b200")
    ref_dir = os.path.join(ROOT, "oracle", "_ref")
    subprocess.run(["g++", "-std=c++20", "-O1", "-I", REF_INC, "-I", nl, "-I",
                    os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "dropin_engine_excerpt.cpp"),
                    "-L", lib_dir, "-lplora", "-L", ref_dir, "-lref",
                    f"-Wl,-rpath,{lib_dir}", f"-Wl,-rpath,{ref_dir}", "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "engine excerpt ok" in out.stdout
