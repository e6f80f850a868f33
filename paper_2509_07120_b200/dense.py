"""Attention inputs and the dense baseline.

``AttentionInputs`` mirrors /root/reference/pkg/src/bsattn/dense.py:20-55
(same validation and ``scale = 1/sqrt(d)`` computed in float64).  Its
tensors live on the GPU; numpy inputs are uploaded once.

``dense_attention`` (dense.py:58-76) is the DENSE BASELINE the block-sparse
kernel is measured against, not part of the product path: it calls the
library SDPA of the installed PyTorch (cuDNN / FlashAttention on sm_100),
which is exactly the "dense cuDNN/FlashAttention-style baseline on the same
GPU" the benchmark reports.  ``dense_attention_map`` (dense.py:79-102) keeps
the reference's size guard.
"""

from __future__ import annotations

import numpy as np
import torch
import torch.nn.functional as F

from . import _native as N

DEFAULT_MAP_ELEMENT_CAP = 2**31


def _as_input(x, name: str, dev, validate: bool):
    if isinstance(x, torch.Tensor):
        t = x
        if t.dtype not in (torch.float32, torch.bfloat16):
            t = t.float()
        if t.device.type != "cuda":
            if validate and not torch.isfinite(t).all():
                raise ValueError(f"{name} contains non-finite values")
            t = t.to(dev)
        return t, False
    a = np.asarray(x, dtype=np.float32)
    if a.ndim == 0:
        raise ValueError(f"{name} must have at least one dimension")
    if min(a.shape) < 1:
        raise ValueError(f"{name} has a zero-sized dimension: {a.shape}")
    if validate and not np.isfinite(a).all():
        raise ValueError(f"{name} contains non-finite values")
    return torch.from_numpy(np.ascontiguousarray(a)).to(dev), True


class AttentionInputs:
    """Per-head query/key/value tensors of shape (heads, tokens, head_dim).

    Like the reference (dense.py:20-55, as_f32 on each of q/k/v) it rejects
    non-finite values; for device tensors the scan is one min/max reduction
    per tensor, skipped with ``validate=False`` by callers that already
    validated.  Mixed dtypes are promoted to fp32 (the reference makes all
    three fp32)."""

    def __init__(self, q, k, v, *, validate: bool = True):
        dev = N.require_cuda()
        self.q, np_in = _as_input(q, "q", dev, validate)
        self.k, _ = _as_input(k, "k", dev, validate)
        self.v, _ = _as_input(v, "v", dev, validate)
        self.numpy_io = np_in
        for name, t in (("q", self.q), ("k", self.k), ("v", self.v)):
            if t.dim() != 3:
                raise ValueError(f"{name} must be (heads, tokens, head_dim), got {tuple(t.shape)}")
            if min(t.shape) < 1:
                raise ValueError(f"{name} has a zero-sized dimension: {tuple(t.shape)}")
            if t.stride(2) != 1:
                setattr(self, name, t.contiguous())
        if not (self.q.shape == self.k.shape == self.v.shape):
            raise ValueError(f"q/k/v shapes differ: {tuple(self.q.shape)}, "
                             f"{tuple(self.k.shape)}, {tuple(self.v.shape)}")
        if not (self.q.device == self.k.device == self.v.device):
            raise ValueError(f"q/k/v live on different devices: {self.q.device}, "
                             f"{self.k.device}, {self.v.device}")
        if not (self.q.dtype == self.k.dtype == self.v.dtype):
            self.q, self.k, self.v = self.q.float(), self.k.float(), self.v.float()
        on_dev = [t for x, t in zip((q, k, v), (self.q, self.k, self.v))
                  if isinstance(x, torch.Tensor) and x.device.type == "cuda"]
        if validate and on_dev:
            if not N.all_finite(*on_dev):
                raise ValueError("q/k/v contain non-finite values")

    @property
    def heads(self) -> int:
        return self.q.shape[0]

    @property
    def tokens(self) -> int:
        return self.q.shape[1]

    @property
    def head_dim(self) -> int:
        return self.q.shape[2]

    @property
    def scale(self) -> float:
        return 1.0 / float(np.sqrt(self.head_dim))


def dense_attention(inp: AttentionInputs, row_chunk: int = 256):
    """Exact dense multi-head attention via the library SDPA (baseline)."""
    del row_chunk  # the library kernel streams internally
    q, k, v = (t.unsqueeze(0) for t in (inp.q, inp.k, inp.v))
    out = F.scaled_dot_product_attention(q, k, v, scale=inp.scale)[0]
    return out.cpu().numpy() if inp.numpy_io else out


def dense_attention_map(inp: AttentionInputs, max_elements: int = DEFAULT_MAP_ELEMENT_CAP):
    """Full post-softmax probabilities (heads, N, N), refused above the cap."""
    h, n, _ = inp.q.shape
    total = h * n * n
    if total > max_elements:
        raise ValueError(
            f"attention map of {total} elements exceeds cap {max_elements}; "
            "raise max_elements only if you have the memory for it")
    s = torch.matmul(inp.q.float(), inp.k.float().transpose(1, 2)) * np.float32(inp.scale)
    p = torch.softmax(s, dim=-1)
    return p.cpu().numpy() if inp.numpy_io else p
