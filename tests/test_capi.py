"""The C-ABI library builds, loads without a GPU and exports exactly the entry points
include/dsv.h declares (CPU only: no kernel is launched)."""

import ctypes
import re
from pathlib import Path

from paper_2502_07590_b200 import _lib

HEADER = Path(__file__).resolve().parent.parent / "include" / "dsv.h"


def _declared():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:int|long long|const char\*)\s+(dsv_\w+)\s*\(", text, re.M)))


def test_header_declares_the_boundary():
    names = _declared()
    for must in ("dsv_topk", "dsv_sparse_fwd", "dsv_sparse_bwd", "dsv_project", "dsv_gemm_bf16",
                 "dsv_scores_f32", "dsv_rows_fwd", "dsv_rows_bwd", "dsv_gather_rows", "dsv_copy_jobs"):
        assert must in names


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    for name in _declared():
        assert hasattr(lib, name), f"{name} missing from libdsv.so"
        assert name in _lib.SIGNATURES, f"{name} has no ctypes signature"
    assert set(_lib.SIGNATURES) == set(_declared())


def test_library_is_loadable_without_a_driver():
    lib = ctypes.CDLL(str(_lib.LIB_PATH))
    lib.dsv_version.restype = ctypes.c_int
    assert lib.dsv_version() >= 100


def test_invalid_arguments_are_reported_not_launched():
    lib = _lib.load()
    # empty shapes are rejected by the boundary before any CUDA call
    rc = lib.dsv_topk(None, 0, 1, 0, None, 1, None, 0, None, None)
    assert rc == _lib.DSV_EINVAL
    assert b"topk" in lib.dsv_last_error()
    rc = lib.dsv_sparse_fwd(None, None, None, None, None, None, 1, None, None, 1, 1, 1, 1, 96,
                            ctypes.c_float(0.1), None, None, None, 0, None, 0, None, 0, None, 0, 0, None)
    assert rc == _lib.DSV_EUNSUPPORTED
