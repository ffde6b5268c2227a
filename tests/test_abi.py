"""CPU-side checks of the boundary: the C-ABI library builds for sm_100a,
loads, and exports every entry point include/gs_render.h declares (no compute
calls: this host has no GPU)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "gs_render.h")


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(gs_[a-z_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib_path():
    from paper_2604_02120_b200 import build
    return build.build()


def test_header_declares_the_north_star_entry_point():
    names = _declared()
    assert "gs_render" in names
    for n in ("gs_ctx_create", "gs_ctx_destroy", "gs_debug_preprocess", "gs_debug_binning",
              "gs_debug_blend", "gs_debug_exponents", "gs_render_views_host"):
        assert n in names


def test_library_exports_every_declared_symbol(lib_path):
    lib = ctypes.CDLL(lib_path)
    for name in _declared():
        assert hasattr(lib, name), name
    from paper_2604_02120_b200 import _binding
    assert sorted(_binding.EXPORTS) == _declared()


def test_exports_are_plain_c_symbols(lib_path):
    out = subprocess.run(["nm", "-D", "--defined-only", lib_path], capture_output=True, text=True).stdout
    syms = {l.split()[-1] for l in out.splitlines() if l.strip()}
    for name in _declared():
        assert name in syms, f"{name} not exported unmangled"


def test_binary_is_sm100a_with_tcgen05(lib_path):
    out = subprocess.run(["cuobjdump", "-sass", lib_path], capture_output=True, text=True).stdout
    assert "sm_100a" in out or "SM100" in out.upper()
    assert "UTCHMMA" in out or "UTCMMA" in out or "UTC" in out, "no tcgen05 MMA in the SASS"
    assert "LDTM" in out, "no tcgen05.ld in the SASS"


def test_binding_refuses_to_run_without_library(tmp_path, monkeypatch):
    from paper_2604_02120_b200 import _binding
    monkeypatch.setattr(_binding, "LIB_PATH", str(tmp_path / "missing.so"))
    monkeypatch.setattr(_binding, "_lib", None)
    with pytest.raises(RuntimeError):
        _binding.load()


def test_product_package_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2604_02120_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dp, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "liboracle" not in txt and "oracle.c" not in txt, f
