"""ctypes binding of libdsv.so (the C ABI in include/dsv.h).

The shared library is the product: every hot-path call goes through it. There
is no CPU fallback — if the library is missing or no CUDA device is present,
the calls raise.
"""

from __future__ import annotations

import ctypes
import os
from ctypes import c_double, c_float, c_int, c_longlong, c_void_p
from pathlib import Path

_PKG = Path(__file__).resolve().parent
# DSV_LIB: an alternate build of the same library (ablation / profiling variants)
LIB_PATH = Path(os.environ["DSV_LIB"]) if os.environ.get("DSV_LIB") else _PKG / "libdsv.so"

DSV_OK, DSV_EINVAL, DSV_EUNSUPPORTED, DSV_ECUDA = 0, 1, 2, 3
DTYPE_F32, DTYPE_BF16, DTYPE_F64 = 0, 1, 2

# name -> argtypes (restype is int unless listed in _RESTYPES)
SIGNATURES = {
    "dsv_version": [],
    "dsv_last_error": [],
    "dsv_device_sm_count": [],
    "dsv_gemm_bf16": [c_void_p, c_longlong, c_longlong, c_void_p, c_longlong, c_longlong,
                      c_void_p, c_int, c_longlong, c_longlong, c_int, c_int, c_int, c_int,
                      c_void_p],
    "dsv_project": [c_void_p, c_void_p, c_void_p, c_int, c_int, c_int, c_void_p],
    "dsv_proxy_scores": [c_void_p, c_longlong, c_longlong, c_void_p, c_longlong, c_longlong,
                         c_void_p, c_longlong, c_longlong, c_int, c_int, c_int, c_int, c_void_p],
    "dsv_scores_f32": [c_void_p, c_longlong, c_longlong, c_void_p, c_longlong, c_longlong,
                       c_void_p, c_longlong, c_longlong, c_int, c_int, c_int, c_int, c_int,
                       c_void_p],
    "dsv_select_fused": [c_void_p, c_longlong, c_longlong, c_void_p, c_longlong, c_longlong, c_int,
                         c_int, c_int, c_int, c_void_p, c_void_p, c_longlong, c_void_p, c_int,
                         c_void_p, c_longlong, c_void_p],
    "dsv_select_fused_workspace_size": [c_int, c_int, c_int, c_int, c_int],
    "dsv_select_fused_max_clusters": [c_int],
    "dsv_topk": [c_void_p, c_longlong, c_int, c_int, c_void_p, c_int, c_void_p, c_longlong,
                 c_void_p, c_void_p],
    "dsv_sparse_fwd": [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_longlong,
                       c_void_p, c_void_p, c_int, c_int, c_int, c_int, c_int, c_float, c_void_p,
                       c_void_p, c_void_p, c_longlong, c_void_p, c_longlong, c_void_p, c_int,
                       c_void_p, c_int, c_int, c_void_p],
    "dsv_sparse_bwd": [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                       c_void_p, c_void_p, c_longlong, c_void_p, c_void_p, c_int, c_int, c_int,
                       c_int, c_int, c_float, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                       c_int, c_void_p, c_int, c_int, c_void_p],
    "dsv_sparse_bwd_convert": [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                               c_void_p, c_void_p, c_void_p, c_longlong, c_void_p, c_void_p,
                               c_int, c_int, c_int, c_int, c_int, c_float, c_void_p, c_void_p,
                               c_void_p, c_void_p, c_void_p, c_int, c_void_p, c_int, c_int,
                               c_void_p, c_void_p, c_void_p, c_int, c_int, c_void_p, c_void_p],
    "dsv_rows_fwd": [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_int, c_int, c_int,
                     c_int, c_float, c_int, c_void_p, c_void_p, c_void_p],
    "dsv_rows_bwd": [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                     c_void_p, c_int, c_int, c_int, c_int, c_float, c_int, c_void_p, c_void_p,
                     c_void_p, c_void_p],
    "dsv_debug_timeline": [c_void_p, c_int],
    "dsv_debug_select_timeline": [c_void_p, c_int],
    "dsv_copy_jobs": [c_void_p, c_int, c_int, c_void_p],
    "dsv_copy_jobs_threads": [c_void_p, c_int, c_int, c_int, c_void_p],
    "dsv_pred_pass": [c_int, c_void_p, c_void_p, c_void_p, c_int, c_longlong, c_int, c_int, c_int,
                      c_void_p, c_void_p, c_void_p],
    "dsv_varint_index_bytes": [c_void_p, c_longlong, c_void_p, c_int, c_int, c_void_p, c_void_p, c_void_p],
    "dsv_varint_encode": [c_void_p, c_longlong, c_void_p, c_int, c_int, c_void_p, c_void_p, c_void_p,
                          c_void_p],
    "dsv_critical_counts": [c_void_p, c_longlong, c_int, c_int, ctypes.c_double, ctypes.c_double,
                            c_void_p, c_void_p],
    "dsv_scp_pull": [c_void_p, c_int, c_int, c_int, c_int, c_void_p, c_void_p, c_void_p, c_void_p,
                     c_int, c_void_p, c_void_p],
    "dsv_scp_push": [c_void_p, c_int, c_int, c_int, c_int, c_void_p, c_void_p, c_void_p, c_void_p,
                     c_int, c_void_p],
    "dsv_peer_alloc": [c_longlong, c_void_p, c_void_p],
    "dsv_peer_open": [c_void_p, c_void_p],
    "dsv_peer_close": [c_void_p],
    "dsv_peer_free": [c_void_p],
    "dsv_peer_barrier": [c_void_p, c_void_p, c_void_p, c_int, c_int, c_void_p],
    "dsv_gather_rows": [c_void_p, c_longlong, c_void_p, c_int, c_int, c_void_p, c_longlong,
                        c_void_p],
    "dsv_f32_to_bf16": [c_void_p, c_void_p, c_longlong, c_void_p],
    "dsv_f32_to_bf16_rows": [c_void_p, c_int, c_int, c_int, c_void_p, c_int, c_int, c_void_p],
    "dsv_ring_lse_merge": [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_longlong, c_int,
                           c_int, c_void_p, c_void_p],
    "dsv_ring_accum_bf16": [c_void_p, c_void_p, c_longlong, c_int, c_void_p, c_void_p],
    "dsv_ring_accum_f32": [c_void_p, c_void_p, c_longlong, c_int, c_void_p],
    # reference-precision (fp64) path
    "dsv_gemm_f64": [c_void_p, c_longlong, c_longlong, c_longlong, c_void_p, c_longlong, c_longlong,
                     c_longlong, c_void_p, c_longlong, c_longlong, c_int, c_int, c_int, c_int,
                     c_double, c_void_p],
    "dsv_softmax_rows_f64": [c_void_p, c_longlong, c_int, c_int, c_void_p],
    "dsv_topk_f64": [c_void_p, c_longlong, c_int, c_int, c_void_p, c_int, c_void_p, c_longlong,
                     c_void_p, c_void_p],
    "dsv_rows_fwd_f64": [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_int, c_int, c_int,
                         c_int, c_int, c_double, c_void_p, c_void_p, c_void_p],
    "dsv_rows_bwd_f64": [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                         c_void_p, c_int, c_int, c_int, c_int, c_int, c_double, c_void_p, c_void_p,
                         c_void_p, c_void_p],
    "dsv_sorted_stats_scratch_bytes": [c_int, c_int],
    "dsv_sorted_stats_f64": [c_void_p, c_longlong, c_int, c_int, c_double, c_double, c_int,
                             c_void_p, c_void_p, c_void_p, c_longlong, c_void_p],
    "dsv_histogram_f64": [c_void_p, c_longlong, c_int, c_int, c_void_p, c_int, c_void_p, c_void_p],
    "dsv_set_stats_f64": [c_void_p, c_longlong, c_int, c_void_p, c_void_p, c_void_p, c_void_p,
                          c_void_p, c_void_p, c_void_p, c_void_p],
}
_RESTYPES = {"dsv_last_error": ctypes.c_char_p, "dsv_sorted_stats_scratch_bytes": c_longlong,
             "dsv_select_fused_workspace_size": c_longlong}

_lib = None


class DSVError(RuntimeError):
    """A CUDA-side failure reported by libdsv (status DSV_ECUDA / DSV_EUNSUPPORTED)."""


def load(build_if_missing: bool = True) -> ctypes.CDLL:
    """Load (building first if needed and possible) the in-tree libdsv.so."""
    global _lib
    if _lib is not None:
        return _lib
    if build_if_missing and os.environ.get("DSV_NO_BUILD") != "1":
        from . import build as _build
        try:
            if not _build.up_to_date():
                _build.build()
        except RuntimeError:
            if not LIB_PATH.exists():
                raise
    if not LIB_PATH.exists():
        raise DSVError(f"{LIB_PATH} is missing: build it with `python -m paper_2502_07590_b200.build`")
    lib = ctypes.CDLL(str(LIB_PATH))
    for name, args in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = _RESTYPES.get(name, c_int)
    _lib = lib
    return lib


def check(status: int, what: str) -> None:
    if status == DSV_OK:
        return
    msg = load().dsv_last_error().decode(errors="replace")
    if status == DSV_EINVAL:
        raise ValueError(f"{what}: {msg}")
    raise DSVError(f"{what} failed (status {status}): {msg}")


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args), name)
