"""Elementary numerics on the device and the .bsat tensor file format.

* ``row_softmax`` (reference tensorio.py:73-87) is the softmax of the pooled
  scores. It is on the hot path and runs in libbsa.so, bit-exact with the
  reference's numpy arithmetic.
* ``as_f32`` / ``read_tensor`` / ``write_tensor`` (tensorio.py:47-59,
  :90-141) are the host-side plumbing of the ``mask`` / ``attend`` CLI
  flows. They keep the reference's byte layout and
  error classes, so files written by either package load in the other:

      "BSAT" | u32 version = 1 | u8 dtype = 0 (f32) | u32 ndim | ndim x u64 dims
      | float32 payload, row-major, little-endian
"""

from __future__ import annotations

import struct

import numpy as np
import torch

from . import _native as N
from .maskpred import _out, _to_device

MAGIC = b"BSAT"
VERSION = 1
DTYPE_F32 = 0
_HEAD = struct.Struct("<4sIBI")


class TensorFileError(ValueError):
    """A .bsat file could not be decoded."""


class BadMagicError(TensorFileError):
    pass


class UnsupportedDTypeError(TensorFileError):
    pass


class TruncatedPayloadError(TensorFileError):
    pass


def as_f32(x, name: str = "tensor") -> np.ndarray:
    """C-contiguous float32 copy-or-view of ``x``; rejects zero-sized
    dimensions and non-finite entries (ValueError)."""
    a = np.ascontiguousarray(x, dtype=np.float32)
    if a.ndim == 0:
        raise ValueError(f"{name} must have at least one dimension")
    if 0 in a.shape:
        raise ValueError(f"{name} has a zero-sized dimension: {a.shape}")
    if not np.isfinite(a).all():
        raise ValueError(f"{name} contains non-finite values")
    return a


def write_tensor(path, t) -> None:
    """Write a float32 tensor (numpy array or torch tensor) as .bsat."""
    if isinstance(t, torch.Tensor):
        t = t.detach().float().cpu().numpy()
    a = as_f32(t)
    with open(path, "wb") as f:
        f.write(_HEAD.pack(MAGIC, VERSION, DTYPE_F32, a.ndim))
        f.write(struct.pack(f"<{a.ndim}Q", *a.shape))
        f.write(a.astype("<f4", copy=False).tobytes())


def read_tensor(path) -> np.ndarray:
    """Decode a .bsat file into a fresh float32 array, or raise the
    TensorFileError subclass naming what is wrong (never a partial tensor)."""
    with open(path, "rb") as f:
        raw = f.read()
    if len(raw) < _HEAD.size:
        raise TruncatedPayloadError(f"file too short for header: {len(raw)} bytes")
    magic, version, dtype, ndim = _HEAD.unpack_from(raw)
    if magic != MAGIC:
        raise BadMagicError(f"bad magic {magic!r}, expected {MAGIC!r}")
    if version != VERSION:
        raise TensorFileError(f"unsupported version {version}")
    if dtype != DTYPE_F32:
        raise UnsupportedDTypeError(f"unsupported dtype code {dtype}")
    if ndim < 1:
        raise TensorFileError("ndim must be >= 1")
    body = _HEAD.size + 8 * ndim
    if len(raw) < body:
        raise TruncatedPayloadError("file too short for dims")
    shape = struct.unpack_from(f"<{ndim}Q", raw, _HEAD.size)
    if 0 in shape:
        raise TensorFileError(f"zero-sized dimension in {shape}")
    count = int(np.prod(shape, dtype=np.int64))
    end = body + 4 * count
    if len(raw) < end:
        raise TruncatedPayloadError(
            f"payload truncated: have {len(raw) - body} bytes, need {4 * count}")
    if len(raw) > end:
        raise TensorFileError(f"{len(raw) - end} trailing bytes after payload")
    t = np.frombuffer(raw, dtype="<f4", count=count, offset=body).astype(np.float32).reshape(shape)
    if not np.isfinite(t).all():
        raise TensorFileError("payload contains non-finite values")
    return t


def row_softmax(a, scale: float = 1.0):
    """Row-wise softmax of ``scale * a`` with subtract-max stabilisation,
    bit-exact with the reference's numpy arithmetic."""
    t, was_np = _to_device(a, "a", allow_bf16=False)
    if t.dim() != 2:
        raise ValueError(f"row_softmax expects a 2-D input, got shape {tuple(t.shape)}")
    t = t.contiguous()
    out = torch.empty_like(t)
    L = N.lib()
    ws = N.workspace(L.bsa_row_softmax_workspace(t.shape[0], t.shape[1]), t.device)
    N.check(L.bsa_row_softmax(t.data_ptr(), t.shape[0], t.shape[1], float(np.float32(scale)),
                              out.data_ptr(), ws.data_ptr(), ws.numel(), N.stream_ptr()),
            "row_softmax")
    return _out(out, was_np)
