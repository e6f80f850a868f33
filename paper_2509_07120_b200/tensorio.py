"""Elementary numerics on the device (tensorio.py:73-87 of the reference).

Only ``row_softmax`` is on the hot path (it is the softmax of the pooled
scores); the reference's .bsat file format is artifact plumbing and out of
scope.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _native as N
from .maskpred import _out, _to_device


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
