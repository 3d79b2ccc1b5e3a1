"""The C ABI library loads and exports every symbol include/igacd.h declares (no GPU needed)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "igacd.h")
LIB = os.path.join(ROOT, "paper_1805_10058_b200", "lib", "libigacd.so")


def declared():
    src = open(HDR).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(igacd_\w+)\s*\(", src, re.M)))


def test_header_declares_the_north_star_calls():
    names = declared()
    for must in ["igacd_create", "igacd_apply", "igacd_vcycle", "igacd_solve", "igacd_destroy",
                 "igacd_restrict", "igacd_prolong", "igacd_smooth", "igacd_residual"]:
        assert must in names


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(LIB):
        import __graft_entry__
        __graft_entry__.build()
    return ctypes.CDLL(LIB)


def test_library_exports_every_declared_symbol(lib):
    missing = [n for n in declared() if not hasattr(lib, n)]
    assert not missing, missing


def test_version_and_argument_errors_without_gpu(lib):
    lib.igacd_version.restype = ctypes.c_char_p
    assert b"sm_100a" in lib.igacd_version()
    lib.igacd_last_error.restype = ctypes.c_char_p
    h = ctypes.c_void_p()
    b0 = (ctypes.c_double * 3)(1, 0, 0)
    # invalid dimension / degree are rejected before any device work
    assert lib.igacd_create(ctypes.byref(h), 4, 2, 8, ctypes.c_double(1), ctypes.c_double(0.1),
                            ctypes.c_double(1), b0, 0, 1, 1, None) == -1
    assert b"dim" in lib.igacd_last_error()
    assert lib.igacd_create(ctypes.byref(h), 2, 9, 8, ctypes.c_double(1), ctypes.c_double(0.1),
                            ctypes.c_double(1), b0, 0, 1, 1, None) == -1
    assert lib.igacd_apply(None, 0, None, None, None) == -1
    assert lib.igacd_destroy(None) == 0


def test_binding_names_match_header():
    import paper_1805_10058_b200.igacd as ig
    for n in declared():
        if n in ("igacd_last_error",):
            continue
        assert hasattr(ig, n), n
