"""CPU-side checks of the boundary: libpac.so loads and exports every symbol that
include/pac.h declares; the binding refuses to run without the library (no fallback);
argument validation needs no GPU."""
import ctypes
import os
import re
import subprocess

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "pac.h")
LIB = os.path.join(ROOT, "paper_2603_15023_b200", "libpac.so")


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(pac_[a-z_0-9]+)\s*\(", src)))


@pytest.fixture(scope="module")
def built():
    import build
    build.build_cuda("libpac")
    return LIB


def test_header_declares_the_boundary_calls():
    names = _declared()
    for need in ("pac_mask", "pac_agg_grouped", "pac_finalize", "pac_posterior_update",
                 "pac_session_create", "pac_session_destroy"):
        assert need in names


def test_library_exports_every_declared_symbol(built):
    out = subprocess.run(["nm", "-D", "--defined-only", built], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (pac_[a-z_0-9]+)", out))
    missing = [n for n in _declared() if n not in exported]
    assert not missing, missing
    L = ctypes.CDLL(built)
    for n in _declared():
        assert hasattr(L, n)


def test_binding_signatures_cover_header(built):
    from paper_2603_15023_b200 import _lib
    assert sorted(_lib.exported_symbols()) == _declared()
    _lib.lib()


def test_library_is_sm100a(built):
    out = subprocess.run(["cuobjdump", "--list-elf", built], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_argument_validation_without_gpu(built):
    from paper_2603_15023_b200 import _lib
    L = _lib.lib()
    # invalid arguments are rejected before any CUDA call
    assert L.pac_mask(None, 10, 0, None, None) == _lib.PAC_E_INVAL
    assert L.pac_mask(None, -1, 0, None, None) == _lib.PAC_E_INVAL
    nb = ctypes.c_size_t()
    assert L.pac_agg_workspace_size(None, 0, 10, ctypes.byref(nb)) == _lib.PAC_E_INVAL
    specs = (_lib.AggSpec * 3)()
    specs[0].kind, specs[1].kind, specs[2].kind = _lib.COUNT, _lib.SUM_I64, 9
    specs[1].d_values = 1234
    assert L.pac_agg_workspace_size(specs, 3, 10, ctypes.byref(nb)) == _lib.PAC_E_INVAL
    assert L.pac_agg_workspace_size(specs, 2, 10, ctypes.byref(nb)) == _lib.PAC_OK and nb.value > 0
    # both mask sources / neither -> INVAL
    t = _lib.Table()
    assert L.pac_agg_grouped(None, None, 0, None, 0, specs, 2, 10, ctypes.byref(t), 10, None, 0, None) \
        == _lib.PAC_E_INVAL
    assert L.pac_session_create(1, -1.0, ctypes.byref(ctypes.c_void_p())) == _lib.PAC_E_INVAL
    assert L.pac_posterior_update(None, None, 0.0, 1.0, None) == _lib.PAC_E_INVAL
    assert "sm_100a" in L.pac_version().decode()


def test_product_package_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2603_15023_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in txt.replace("oracle/", "").lower() or f.endswith(".cu"), f
                assert "import oracle" not in txt and "from oracle" not in txt, f
