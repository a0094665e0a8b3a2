"""The C-ABI library loads without a GPU and exports every entry point that
include/ssfm.h declares (no compute calls here)."""
import ctypes as ct
import os
import re

from paper_2510_13310_b200 import _native

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "ssfm.h")


def declared_functions():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(ssfm_[a-z_0-9]+)\s*\(", text)))


def test_header_declares_expected_entry_points():
    decl = declared_functions()
    assert set(_native.EXPORTS) <= set(decl)
    assert "ssfm_lm_solve" in decl and "ssfm_create_ba" in decl and "ssfm_create_gp" in decl


def test_library_exports_every_declared_symbol():
    lib = _native.load()
    for name in declared_functions():
        assert hasattr(lib, name), name
    assert lib.ssfm_version().decode().startswith("ssfm-b200")


def test_struct_layouts_match_header_sizes():
    # field counts / packing of the ctypes mirrors
    assert ct.sizeof(_native.IterRecordC) == 4 * 4 + 3 * 8 + 8 + 8
    assert ct.sizeof(_native.LMConfigC) == 8 * 10
    assert _native.BADescC.cam_idx.offset == 40


def test_invalid_arguments_rejected_without_gpu_work():
    lib = _native.load()
    out = ct.c_void_p(0)
    rc = lib.ssfm_create_ba(None, None, ct.byref(out))
    assert rc == 9
    assert b"null" in lib.ssfm_last_error()


def test_schur_plan_struct_matches_header():
    # ssfm_schur_plan: 8 int64 sizes then 34 device pointers, header order
    assert ct.sizeof(_native.SchurPlanC) == 8 * 8 + 34 * 8
    text = open(HEADER).read()
    body = text[text.index("typedef struct {\n  int64_t n_params, n_ret"):text.index("} ssfm_schur_plan;")]
    names = re.findall(r"\*\s*([a-z_0-9]+);", body)
    assert tuple(names) == tuple(n for n, _ in _native.SCHUR_PLAN_ARRAYS)
