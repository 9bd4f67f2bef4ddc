"""Argument coercion shared by the reference-compatible API.

Mirrors the reference's validation contract (pkg/src/dynsparse/validate.py:10-25
`as_matrix`): inputs must be 2-D (per head) and finite, otherwise ValueError.
Host inputs (numpy / lists) are moved to the CUDA device; results go back to
the caller's world (numpy in -> numpy out, torch in -> torch out).
"""

from __future__ import annotations

import numpy as np
import torch


class NumericalError(Exception):
    """A computation produced a non-finite result (validate.py:6-7)."""


def device() -> torch.device:
    if not torch.cuda.is_available():
        from ._lib import DSVError

        raise DSVError("the DSV kernels need a CUDA device; there is no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def is_torch(x) -> bool:
    return isinstance(x, torch.Tensor)


def as_matrix(name: str, x, dtype=None):
    """validate.py:10-25 — 2-D, finite; float32 kept, anything else float64."""
    if is_torch(x):
        if x.dim() != 2:
            raise ValueError(f"{name} must be 2D, got shape {tuple(x.shape)}")
        if not bool(torch.isfinite(x).all()):
            raise ValueError(f"{name} contains NaN or Inf")
        return x
    arr = np.asarray(x)
    if dtype is not None:
        arr = arr.astype(dtype, copy=False)
    elif arr.dtype not in (np.float32, np.float64):
        arr = arr.astype(np.float64)
    if arr.ndim != 2:
        raise ValueError(f"{name} must be 2D, got shape {arr.shape}")
    if not np.all(np.isfinite(arr)):
        raise ValueError(f"{name} contains NaN or Inf")
    return arr


def check_same_cols(name_a, a, name_b, b) -> None:
    if a.shape[1] != b.shape[1]:
        raise ValueError(f"{name_a} and {name_b} must share the inner dimension: "
                         f"{a.shape[1]} != {b.shape[1]}")


def to_device(x, dtype: torch.dtype) -> torch.Tensor:
    dev = device()
    if is_torch(x):
        return x.to(device=dev, dtype=dtype).contiguous()
    return torch.from_numpy(np.ascontiguousarray(x)).to(device=dev, dtype=dtype)


def back(t: torch.Tensor, like, np_dtype=None):
    """Return `t` in the caller's world: numpy (with np_dtype) if `like` is host data."""
    if is_torch(like):
        return t
    out = t.detach().cpu().numpy()
    return out.astype(np_dtype, copy=False) if np_dtype is not None else out


def wants_f64(x) -> bool:
    """The reference-precision path: host (numpy) data and torch float64 tensors compute in
    fp64 on the device, like the reference computes in the caller's dtype (float64 by
    default; float32 inputs get fp64 arithmetic and fp32 results). torch fp32 / bf16
    tensors keep the fp32 / tensor-core paths."""
    return (not is_torch(x)) or x.dtype == torch.float64


def result_dtype(*xs):
    """numpy result dtype of the reference's arithmetic on host inputs (None for torch)."""
    if any(is_torch(x) for x in xs):
        return None
    return np.result_type(*[np.asarray(x).dtype for x in xs])


def check_unit_interval(name: str, value: float, *, open_low=False, open_high=False) -> float:
    """validate.py:36-44."""
    value = float(value)
    low_ok = value > 0.0 if open_low else value >= 0.0
    high_ok = value < 1.0 if open_high else value <= 1.0
    if not (low_ok and high_ok and np.isfinite(value)):
        lo = "(" if open_low else "["
        hi = ")" if open_high else "]"
        raise ValueError(f"{name} must lie in {lo}0, 1{hi}, got {value}")
    return value
