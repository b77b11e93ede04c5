"""The C-ABI library builds, loads and exports every symbol include/sip.h
declares; argument validation works without a GPU (no compute calls)."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "sip.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sip_[a-z_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def L():
    from paper_1902_09699_b200 import build as b
    b.build()
    import paper_1902_09699_b200 as pkg
    return pkg.lib()


def test_header_declares_boundary_calls():
    syms = declared_symbols()
    for name in ("sip_create_grid", "sip_add_set", "sip_project", "sip_project_multilevel",
                 "sip_set_option", "sip_destroy"):
        assert name in syms


def test_library_exports_every_declared_symbol(L):
    import paper_1902_09699_b200 as pkg
    syms = declared_symbols()
    assert sorted(pkg.EXPORTS) == syms
    for name in syms:
        assert hasattr(L, name), name


def test_library_targets_sm100a_only():
    lib = os.path.join(ROOT, "paper_1902_09699_b200", "libsip.so")
    out = os.popen(f"/usr/local/cuda/bin/cuobjdump --list-elf {lib} 2>&1").read()
    assert "sm_100a" in out
    assert "sm_90" not in out and "sm_80" not in out


def test_status_strings(L):
    for s in (0, 1, -1, -2, -3, -4, -5, -6, -7, -8, -9):
        assert len(L.sip_status_string(s)) > 0


def test_argument_validation_without_gpu(L):
    out = C.c_void_p()
    n = (C.c_int64 * 2)(8, 8)
    assert L.sip_create_grid(4, n, None, 0, None, None, C.byref(out)) == -1      # bad ndim
    assert L.sip_create_grid(2, n, None, 7, None, None, C.byref(out)) == -1      # bad dtype
    n1 = (C.c_int64 * 2)(1, 8)
    assert L.sip_create_grid(2, n1, None, 0, None, None, C.byref(out)) == -4     # n < 2
    hbad = (C.c_double * 2)(1.0, -1.0)
    assert L.sip_create_grid(2, n, hbad, 0, None, None, C.byref(out)) == -3      # h <= 0
    assert L.sip_project(None, None, None, 10, 1e-3, None) == -1
    assert L.sip_add_set(None, 0, None, 0, None, None) == -1
    assert L.sip_set_option(None, b"rho0", C.c_double(1.0)) == -1
    L.sip_destroy(None)
