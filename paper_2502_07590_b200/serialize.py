"""Index-set memory and wire formats.

Reference: pkg/src/dynsparse/serialize.py:99-151 and dispatcher.py:135-137. Same names and
byte-for-byte output:
  * raw_index_payload(indices, index_width)  fixed-width rows back to back; its size is
    `index_memory_bytes(S, k, width)` for uniform k (the dispatcher's memory model);
  * encode_index_sets(indices)               varint(n_rows), per row varint(count) and the
    varint deltas of the strictly increasing indices;
  * decode_index_sets(raw)                   the inverse (host).
Device index sets — the layer's `SelectedKV` (int32 [H, G, k_max] + counts) or any int32
[rows, k_max] tensor with per-row counts — are encoded on the GPU (dsv_varint_index_bytes
/ dsv_varint_encode, one warp per row) and `offload` moves the encoded bytes to pinned host
memory asynchronously (c5: ~2.6 GB of int32 index sets per rank shrink to their ~1-2-byte
varint deltas before crossing PCIe).
"""

from __future__ import annotations

import io

import numpy as np
import torch

from . import _lib


def index_memory_bytes(s_total: int, k: int, index_width: int = 4) -> int:
    """Bytes for per-query index buffers; matches the raw payload (dispatcher.py:135-137)."""
    return s_total * k * index_width


def _rows(indices):
    return indices.indices if hasattr(indices, "indices") else indices


def raw_index_payload(indices, index_width: int = 4) -> bytes:
    """Fixed-width payload (serialize.py:99-107)."""
    dtype = {4: np.int32, 8: np.int64}.get(index_width)
    if dtype is None:
        raise ValueError("index_width must be 4 or 8")
    out = io.BytesIO()
    for row in _rows(indices):
        out.write(np.ascontiguousarray(np.asarray(row, dtype=dtype)).tobytes())
    return out.getvalue()


def _varint(v: int) -> bytes:
    out = bytearray()
    while True:
        b = v & 0x7F
        v >>= 7
        if v:
            out.append(b | 0x80)
        else:
            out.append(b)
            return bytes(out)


def encode_device(idx: torch.Tensor, counts=None) -> torch.Tensor:
    """Varint-delta encoding of a device int32 [rows, k_max] index tensor (row r valid up to
    counts[r], or all k_max columns) -> uint8 device tensor with the reference's bytes."""
    if not idx.is_cuda or idx.dtype != torch.int32 or idx.dim() != 2 or idx.stride(1) != 1:
        raise ValueError("encode_device expects a CUDA int32 [rows, k_max] tensor with unit column stride")
    rows, kmax = idx.shape
    dev = idx.device
    st = torch.cuda.current_stream().cuda_stream
    cnt = None
    if counts is not None:
        cnt = torch.as_tensor(counts, dtype=torch.int32, device=dev).contiguous().reshape(-1)
        if cnt.numel() != rows:
            raise ValueError("counts must have one entry per row")
        if bool((cnt < 0).any()) or bool((cnt > kmax).any()):
            raise ValueError("counts must lie in [0, k_max]")
    err = torch.zeros((1,), dtype=torch.int32, device=dev)
    lens = torch.empty((rows,), dtype=torch.int64, device=dev)
    cptr = cnt.data_ptr() if cnt is not None else 0
    _lib.call("dsv_varint_index_bytes", idx.data_ptr(), idx.stride(0), cptr, kmax, rows,
              lens.data_ptr(), err.data_ptr(), st)
    header = _varint(rows)
    off = torch.cumsum(lens, 0) - lens + len(header)
    total = len(header) + int(lens.sum().item())
    if int(err.item()) & 1:
        raise ValueError("varints are unsigned")
    if int(err.item()) & 2:
        raise ValueError("index rows must be strictly increasing")
    out = torch.empty((total,), dtype=torch.uint8, device=dev)
    out[: len(header)] = torch.tensor(list(header), dtype=torch.uint8, device=dev)
    _lib.call("dsv_varint_encode", idx.data_ptr(), idx.stride(0), cptr, kmax, rows, off.data_ptr(),
              out.data_ptr(), err.data_ptr(), st)
    return out


def encode_index_sets(indices) -> bytes:
    """Varint-delta encoding of sorted per-query index lists (serialize.py:119-135).
    Device SelectedKV / int32 tensors are encoded on the GPU; lists on the host."""
    if isinstance(indices, torch.Tensor) and indices.is_cuda:
        return encode_device(indices.reshape(-1, indices.shape[-1]).contiguous()).cpu().numpy().tobytes()
    if hasattr(indices, "idx") and hasattr(indices, "kcount"):     # layer.SelectedKV
        H, G, kmax = indices.idx.shape
        counts = indices.kcount.to(torch.int32)[:, None].expand(H, G).reshape(-1)
        return encode_device(indices.idx.reshape(H * G, kmax), counts).cpu().numpy().tobytes()
    rows = _rows(indices)
    out = bytearray(_varint(len(rows)))
    for row in rows:
        row = np.asarray(row, dtype=np.int64)
        out += _varint(row.size)
        prev = 0
        for j, value in enumerate(row):
            delta = int(value) if j == 0 else int(value) - prev
            if delta < 0 or (j > 0 and delta == 0):
                raise ValueError("index rows must be strictly increasing")
            out += _varint(delta)
            prev = int(value)
    return bytes(out)


def decode_index_sets(raw: bytes) -> list:
    """Inverse of encode_index_sets (serialize.py:138-151)."""
    def rd(pos):
        result, shift = 0, 0
        while True:
            b = raw[pos]
            pos += 1
            result |= (b & 0x7F) << shift
            if not b & 0x80:
                return result, pos
            shift += 7
    n_rows, pos = rd(0)
    rows = []
    for _ in range(n_rows):
        count, pos = rd(pos)
        values = np.empty(count, dtype=np.int64)
        prev = 0
        for j in range(count):
            delta, pos = rd(pos)
            prev = delta if j == 0 else prev + delta
            values[j] = prev
        rows.append(values)
    return rows


def offload(encoded: torch.Tensor, stream=None):
    """Asynchronous copy of an encoded device buffer to pinned host memory on `stream`
    (default: a side stream). Returns (host tensor, event to wait on before reading)."""
    stream = stream or torch.cuda.Stream(device=encoded.device)
    host = torch.empty(encoded.shape, dtype=encoded.dtype, pin_memory=True)
    stream.wait_stream(torch.cuda.current_stream(encoded.device))
    with torch.cuda.stream(stream):
        host.copy_(encoded, non_blocking=True)
        ev = torch.cuda.Event()
        ev.record(stream)
    encoded.record_stream(stream)
    return host, ev


# ---- binary tensors (serialize.py:1-85 "DTSR" layout), used by predictor checkpoints.
# Little-endian: b"DTSR", version 1, dtype code (1 f64, 2 f32, 3 i32, 4 i64), ndim (1..4), a
# reserved zero byte, ndim uint64 sizes, then the C-order element data.
MAGIC = b"DTSR"
VERSION = 1
_CODES = {np.dtype(np.float64): 1, np.dtype(np.float32): 2, np.dtype(np.int32): 3,
          np.dtype(np.int64): 4}
_DTYPES = {c: dt for dt, c in _CODES.items()}


def canonical_json(obj) -> str:
    """Sorted keys, compact separators, trailing newline (serialize.py:36-38)."""
    import json

    return json.dumps(obj, sort_keys=True, separators=(",", ":")) + "\n"


def tensor_bytes(arr) -> bytes:
    arr = np.ascontiguousarray(arr)
    if arr.dtype not in _CODES:
        raise ValueError(f"unsupported dtype {arr.dtype}")
    if not 1 <= arr.ndim <= 4:
        raise ValueError(f"unsupported rank {arr.ndim}")
    head = MAGIC + bytes([VERSION, _CODES[arr.dtype], arr.ndim, 0])
    head += np.asarray(arr.shape, dtype="<u8").tobytes()
    return head + arr.astype(arr.dtype.newbyteorder("<"), copy=False).tobytes(order="C")


def tensor_from_bytes(raw: bytes) -> np.ndarray:
    if raw[:4] != MAGIC:
        raise ValueError("bad tensor magic")
    if raw[4] != VERSION:
        raise ValueError(f"unsupported tensor format version {raw[4]}")
    dt = _DTYPES.get(raw[5])
    if dt is None:
        raise ValueError(f"unknown dtype code {raw[5]}")
    ndim = raw[6]
    dims = tuple(int(x) for x in np.frombuffer(raw, dtype="<u8", count=ndim, offset=8))
    return np.frombuffer(raw, dtype=dt.newbyteorder("<"), offset=8 + 8 * ndim).reshape(dims).astype(dt)


def save_tensor(path, arr) -> None:
    with open(path, "wb") as fh:
        fh.write(tensor_bytes(np.asarray(arr)))


def load_tensor(path) -> np.ndarray:
    with open(path, "rb") as fh:
        return tensor_from_bytes(fh.read())
