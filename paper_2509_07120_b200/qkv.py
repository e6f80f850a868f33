"""The step before the path, fused: the QKV projection
of a global-attention block on the tensor cores, with the pooled patch Q/K
the mask predictor needs emitted by the GEMM epilogue.

The reference has no model code; its hot path starts at
``predict_mask(q_patches, k_patches, policy)`` (maskpred.py:177-194), which
pools Q and K per token block (block_pool, maskpred.py:104-120) before
scoring.  Here the projection that produces Q/K writes, in the same pass:

* Q, K, V as (heads, tokens, 64) bf16 in the partitioned token order
  [specials | patches] (layout.py:113-138), which ``sparse_attention(...,
  inputs_permuted=True)`` reads in place (no pack pass);
* the block means of the bf16 patch rows of Q (block_q 128) and K (block_k
  64), bit-identical to ``block_pool`` of those tensors, so
  ``predict_mask_pooled`` gives exactly ``predict_mask``'s mask without
  re-reading Q and K.
"""

from __future__ import annotations

import torch

from . import _native as N
from .layout import BlockGeometry, TokenLayout


def qkv_projection(x: torch.Tensor, weight: torch.Tensor, bias: torch.Tensor | None,
                   heads: int, layout: TokenLayout, geometry: BlockGeometry | None = None,
                   *, pooled: bool = True):
    """x (T, C) bf16 CUDA tensor with rows in partitioned order; weight
    (3C, C) bf16 (nn.Linear layout, [Q | K | V] x C); bias (3C) bf16 or None.

    Returns ``(q, k, v, q_pooled, k_pooled)``: q/k/v (heads, T, 64) bf16 in
    the same row order, the pooled tensors (heads, nq, 64) / (heads, nk, 64)
    fp32 (None when ``pooled=False``).  Needs head_dim 64, C % 256 == 0 and
    the 128/64 block geometry (ValueError otherwise)."""
    N.require_cuda()  # a GPU and libbsa.so, or a loud error (no CPU path)
    if not isinstance(x, torch.Tensor) or x.device.type != "cuda":
        raise ValueError("x must be a CUDA tensor")
    if x.dim() != 2 or x.dtype != torch.bfloat16:
        raise ValueError(f"x must be (tokens, C) bf16, got {tuple(x.shape)} {x.dtype}")
    T, C = x.shape
    if T != layout.total_tokens:
        raise ValueError(f"x has {T} rows, layout describes {layout.total_tokens}")
    if C % heads != 0 or C // heads != 64:
        raise ValueError(f"C={C} must be heads ({heads}) x 64")
    if tuple(weight.shape) != (3 * C, C) or weight.dtype != torch.bfloat16:
        raise ValueError(f"weight must be (3C, C) = ({3 * C}, {C}) bf16, got "
                         f"{tuple(weight.shape)} {weight.dtype}")
    if bias is not None and (tuple(bias.shape) != (3 * C,) or bias.dtype != torch.bfloat16):
        raise ValueError(f"bias must be ({3 * C},) bf16")
    for name, t in (("weight", weight), ("bias", bias)):
        if t is not None and t.device != x.device:
            raise ValueError(f"{name} is on {t.device}, x on {x.device}")
    g = geometry or BlockGeometry(layout.patch_tokens, 128, 64)
    if g.patch_tokens != layout.patch_tokens:
        raise ValueError(f"geometry covers {g.patch_tokens} patch tokens, layout {layout.patch_tokens}")
    x = x.contiguous()
    weight = weight.contiguous()
    bias = bias.contiguous() if bias is not None else None
    H = heads
    q, k, v = (torch.empty((H, T, 64), dtype=torch.bfloat16, device=x.device) for _ in range(3))
    qp = kp = None
    if pooled:
        qp = torch.empty((H, g.nq_blocks, 64), dtype=torch.float32, device=x.device)
        kp = torch.empty((H, g.nk_blocks, 64), dtype=torch.float32, device=x.device)
    with N.on_device(x.device):
        N.check(N.lib().bsa_qkv_project_pooled(
            x.data_ptr(), T, C, weight.data_ptr(), N.ptr(bias), H, 64, layout.special_tokens,
            g.block_q, g.block_k, q.data_ptr(), k.data_ptr(), v.data_ptr(), N.ptr(qp), N.ptr(kp),
            N.stream_ptr()), "qkv_projection")
    return q, k, v, qp, kp


def proj_residual(o: torch.Tensor, weight: torch.Tensor, bias: torch.Tensor | None,
                  residual: torch.Tensor, *, out: torch.Tensor | None = None):
    """The block's output projection with its residual, on the tensor cores:
    ``residual + o' W^T + bias`` with o' the (T, C) token-major view of the
    attention output ``o`` (heads, T, 64) bf16 -- read head-major in place
    as the GEMM's A operand (no transpose pass) -- and one bf16 rounding of
    the fp32 sum.  ``out`` may be ``residual`` itself (in-place update).
    Returns the (T, C) bf16 result."""
    N.require_cuda()
    for name, t in (("o", o), ("weight", weight), ("residual", residual)):
        if not isinstance(t, torch.Tensor) or t.device.type != "cuda" or t.dtype != torch.bfloat16:
            raise ValueError(f"{name} must be a bf16 CUDA tensor")
    if o.dim() != 3 or o.shape[2] != 64:
        raise ValueError(f"o must be (heads, tokens, 64), got {tuple(o.shape)}")
    H, T, _ = o.shape
    C = H * 64
    if tuple(weight.shape) != (C, C):
        raise ValueError(f"weight must be ({C}, {C}), got {tuple(weight.shape)}")
    if tuple(residual.shape) != (T, C):
        raise ValueError(f"residual must be ({T}, {C}), got {tuple(residual.shape)}")
    if bias is not None and (tuple(bias.shape) != (C,) or bias.dtype != torch.bfloat16):
        raise ValueError(f"bias must be ({C},) bf16")
    for name, t in (("weight", weight), ("residual", residual), ("bias", bias)):
        if t is not None and t.device != o.device:
            raise ValueError(f"{name} is on {t.device}, o on {o.device}")
    if out is None:
        out = torch.empty((T, C), dtype=torch.bfloat16, device=o.device)
    elif tuple(out.shape) != (T, C) or out.dtype != torch.bfloat16 or not out.is_contiguous() \
            or out.device != o.device:
        raise ValueError(f"out must be a contiguous ({T}, {C}) bf16 tensor on {o.device}")
    o, weight = o.contiguous(), weight.contiguous()
    if not residual.is_contiguous():
        residual = residual.contiguous()
    bias = bias.contiguous() if bias is not None else None
    with N.on_device(o.device):
        N.check(N.lib().bsa_proj_residual(o.data_ptr(), H, T, weight.data_ptr(), N.ptr(bias),
                                          residual.data_ptr(), out.data_ptr(), N.stream_ptr()),
                "proj_residual")
    return out
