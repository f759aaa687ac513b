"""The C-ABI library loads and exports every symbol include/plora.h declares
(no compute calls: these run without a GPU)."""
import ctypes
import os
import re
import subprocess

from paper_2512_20210_b200 import _native as N

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    with open(os.path.join(ROOT, "include", "plora.h")) as f:
        text = f.read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(plora_[a-z0-9_]+)\s*\(", text)))


def test_header_symbols_exported():
    lib = ctypes.CDLL(N.LIB_PATH)
    names = _declared_symbols()
    assert len(names) > 60
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_python_binding_covers_header():
    assert set(_declared_symbols()) == set(N.EXPORTED)


def test_library_is_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", N.LIB_PATH], capture_output=True, text=True)
    assert "sm_100a" in out.stdout
    assert not re.search(r"sm_(80|86|89|90)\b", out.stdout)


def test_header_compiles_as_c():
    src = os.path.join(ROOT, "include", "plora.h")
    r = subprocess.run(["gcc", "-std=c99", "-fsyntax-only", "-x", "c", src], capture_output=True,
                       text=True)
    assert r.returncode == 0, r.stderr


def test_no_oracle_in_product():
    """The product never imports, links or loads the oracle."""
    pkg = os.path.join(ROOT, "paper_2512_20210_b200")
    for dirpath, _, files in os.walk(pkg):
        for fn in files:
            if fn.endswith((".py", ".cu", ".cpp", ".hpp", ".h")) or fn == "Makefile":
                with open(os.path.join(dirpath, fn)) as f:
                    body = f.read()
                assert "import oracle" not in body and "from oracle" not in body, fn
                assert "liboracle" not in body and "libref" not in body, fn
    out = subprocess.run(["ldd", N.LIB_PATH], capture_output=True, text=True).stdout
    assert "oracle" not in out and "libref" not in out
