"""The C++ face (include/plora.hpp) compiles against the C ABI and behaves
like lorasim::PagePool (reference tests re-expressed in C++)."""
import os
import subprocess

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
