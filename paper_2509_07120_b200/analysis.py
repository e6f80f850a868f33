"""Dense attention-map statistics on the GPU, without the (H, T, T) map.

SURVEY.md §8f row 4. The reference materialises the post-softmax map
(``dense_attention_map``, /root/reference/pkg/src/bsattn/dense.py:79-102, capped
at 2^31 elements) and reduces it on the CPU (``quadrant_stats``,
analysis.py:47-74). That is what per-layer tau/rho selection tooling needs
(PAPER.md:250-261), but only at small N.

Here S = Q K^T is streamed through the tensor cores twice (libbsa.so,
csrc/bsa_stats_tc.cu):

* ``attention_row_stats``: per query row, the softmax max and the partial
  sums over special and patch keys (and their maxima). Every quadrant
  statistic of the reference is a function of these.
* ``block_attention_map``: the attention mass of every patch q-block on every
  patch k-block, at the BlockMask geometry (128 x 64). This is what the
  pooled-score mask predictor estimates; ``mask_recall`` measures how much of
  it a mask keeps.

q and k enter the tensor cores as bf16 (fp32 inputs are rounded), with fp32
accumulation and MUFU exp2.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from .dense import AttentionInputs
from .layout import TokenLayout, special_token_indices

QUADRANTS = ("S2S", "S2P", "P2S", "P2P")


@dataclass(frozen=True)
class QuadrantStats:
    """Per-head mean/max attention per quadrant (analysis.py:22-44).

    ``means`` and ``maxes`` map quadrant name to a (heads,) float64 array;
    quadrants empty for the layout (no special tokens) are absent."""

    means: dict
    maxes: dict
    heads: int

    def aggregate(self) -> dict:
        """Per quadrant: (mean of means, std of means, mean of maxes, std of maxes)."""
        out = {}
        for quad in self.means:
            mn, mx = self.means[quad], self.maxes[quad]
            out[quad] = (float(mn.mean()), float(mn.std()), float(mx.mean()), float(mx.std()))
        return out


def _bf16_qk(inp: AttentionInputs):
    q, k = inp.q, inp.k
    if q.shape[2] != 64:
        raise ValueError(f"attention statistics need head_dim 64, got {q.shape[2]}")
    return (q if q.dtype == torch.bfloat16 else q.to(torch.bfloat16),
            k if k.dtype == torch.bfloat16 else k.to(torch.bfloat16))


def _check_layout(inp: AttentionInputs, layout: TokenLayout):
    if inp.q.shape[1] != layout.total_tokens:
        raise ValueError(f"inputs have {inp.q.shape[1]} tokens but layout describes "
                         f"{layout.total_tokens}")


def _workspace(layout: TokenLayout, heads: int, device):
    L = N.lib()
    return N.workspace(L.bsa_attention_stats_workspace(N.layout_desc(layout), heads), device)


def attention_row_stats(inp: AttentionInputs, layout: TokenLayout) -> torch.Tensor:
    """(H, T, 5) float32 on the device, per query row in source token order,
    with x = s * scale * log2(e) over all T keys: [m = max x,
    sum_special 2^(x-m), sum_patch 2^(x-m), max_special x, max_patch x]."""
    _check_layout(inp, layout)
    q, k = _bf16_qk(inp)
    H, T, _ = q.shape
    out = torch.empty((H, T, 5), dtype=torch.float32, device=q.device)
    ws = _workspace(layout, H, q.device)
    L = N.lib()
    with N.on_device(q.device):
        N.check(L.bsa_attention_row_stats(N.tensor_desc(q), N.tensor_desc(k),
                                          N.layout_desc(layout), float(np.float32(inp.scale)),
                                          out.data_ptr(), ws.data_ptr(), ws.numel(),
                                          N.stream_ptr()), "attention_row_stats")
    return out


def block_attention_map(inp: AttentionInputs, layout: TokenLayout, row_stats=None):
    """(H, nq, nk) float32: mean over the rows of patch q-block qb (128 rows)
    of the summed softmax probabilities over the keys of patch k-block kb (64
    keys), in the partitioned patch order of BlockMask. Rows sum to the
    fraction of attention on patch keys. numpy inputs give a numpy array."""
    _check_layout(inp, layout)
    q, k = _bf16_qk(inp)
    if row_stats is None:
        row_stats = attention_row_stats(inp, layout)
    H, T, _ = q.shape
    Tp = layout.patch_tokens
    nq, nk = -(-Tp // 128), -(-Tp // 64)
    out = torch.empty((H, nq, nk), dtype=torch.float32, device=q.device)
    ws = _workspace(layout, H, q.device)
    L = N.lib()
    with N.on_device(q.device):
        N.check(L.bsa_block_attention_map(N.tensor_desc(q), N.tensor_desc(k),
                                          N.layout_desc(layout), float(np.float32(inp.scale)),
                                          row_stats.data_ptr(), out.data_ptr(), ws.data_ptr(),
                                          ws.numel(), N.stream_ptr()), "block_attention_map")
    return out.cpu().numpy() if inp.numpy_io else out


def _special_mask(layout: TokenLayout, device) -> torch.Tensor:
    sp = torch.zeros(layout.total_tokens, dtype=torch.bool, device=device)
    idx = special_token_indices(layout)
    if len(idx):
        sp[torch.as_tensor(np.asarray(idx), device=device)] = True
    return sp


def quadrant_stats_from_rows(row_stats: torch.Tensor, layout: TokenLayout) -> QuadrantStats:
    """The reference's quadrant_stats (analysis.py:47-74) of the full map,
    from attention_row_stats: the mean over a quadrant is the mean over its
    query rows of the probability mass on its key kind, over the key count;
    the max is max over rows of 2^(x_kind_max - m) / l."""
    rs = row_stats.double()
    m, ls, lp, xs, xp = (rs[..., i] for i in range(5))
    l = ls + lp
    sp = _special_mask(layout, rs.device)
    n_s = int(sp.sum())
    n_p = layout.total_tokens - n_s
    kinds = {"S": (ls / l, torch.exp2(xs - m) / l, n_s), "P": (lp / l, torch.exp2(xp - m) / l, n_p)}
    rows = {"S": sp, "P": ~sp}
    means, maxes = {}, {}
    for quad in QUADRANTS:
        qk, kk = quad[0], quad[2]
        rsel = rows[qk]
        mass, pmax, nkeys = kinds[kk]
        if not bool(rsel.any()) or nkeys == 0:
            continue
        means[quad] = (mass[:, rsel].sum(dim=1) / (int(rsel.sum()) * nkeys)).cpu().numpy()
        maxes[quad] = pmax[:, rsel].amax(dim=1).cpu().numpy()
    return QuadrantStats(means=means, maxes=maxes, heads=int(row_stats.shape[0]))


def quadrant_stats(attn_map, layout: TokenLayout, row_sum_tol: float = 1e-5) -> QuadrantStats:
    """Reduce a materialised (heads, N, N) post-softmax map into per-quadrant
    statistics, as analysis.py:47-74 (same validation and messages), on the
    GPU. For maps too large to materialise use attention_quadrant_stats."""
    dev = N.require_cuda()
    if isinstance(attn_map, torch.Tensor):
        a = attn_map.to(dev, torch.float32)
    else:
        arr = np.asarray(attn_map, dtype=np.float32)
        if arr.ndim == 0 or min(arr.shape) < 1:
            raise ValueError(f"attn_map has a zero-sized dimension: {arr.shape}")
        if not np.isfinite(arr).all():
            raise ValueError("attn_map contains non-finite values")
        a = torch.from_numpy(np.ascontiguousarray(arr)).to(dev)
    if a.dim() != 3 or a.shape[1] != a.shape[2]:
        raise ValueError(f"attn_map must be (heads, N, N), got {tuple(a.shape)}")
    n = layout.total_tokens
    if a.shape[1] != n:
        raise ValueError(f"map covers {a.shape[1]} tokens, layout describes {n}")
    sums = a.sum(dim=2, dtype=torch.float64)
    if float((sums - 1.0).abs().max()) > row_sum_tol:
        raise ValueError("rows do not sum to 1; expected a post-softmax map")
    sp = _special_mask(layout, dev)
    groups = {"S2S": (sp, sp), "S2P": (sp, ~sp), "P2S": (~sp, sp), "P2P": (~sp, ~sp)}
    means, maxes = {}, {}
    for quad, (qsel, ksel) in groups.items():
        if not bool(qsel.any()) or not bool(ksel.any()):
            continue
        sub = a[:, qsel][:, :, ksel]
        means[quad] = sub.double().mean(dim=(1, 2)).cpu().numpy()
        maxes[quad] = sub.amax(dim=(1, 2)).double().cpu().numpy()
    return QuadrantStats(means=means, maxes=maxes, heads=int(a.shape[0]))


def attention_quadrant_stats(inp: AttentionInputs, layout: TokenLayout) -> QuadrantStats:
    """quadrant_stats(dense_attention_map(inp), layout) without the map."""
    return quadrant_stats_from_rows(attention_row_stats(inp, layout), layout)


def mask_recall(block_map, mask) -> np.ndarray | torch.Tensor:
    """Per (head, q-block): the fraction of the patch-key attention mass that
    the mask's selected k-blocks keep (1.0 for a full mask)."""
    a = block_map if isinstance(block_map, torch.Tensor) else torch.from_numpy(
        np.asarray(block_map, dtype=np.float32))
    sel = torch.from_numpy(np.asarray(mask.blocks)).to(a.device)
    if tuple(sel.shape) != tuple(a.shape):
        raise ValueError(f"mask {tuple(sel.shape)} and block map {tuple(a.shape)} differ")
    a = a.double()
    r = (a * sel).sum(dim=2) / a.sum(dim=2)
    return r if isinstance(block_map, torch.Tensor) else r.cpu().numpy()


__all__ = ["QuadrantStats", "QUADRANTS", "attention_row_stats", "block_attention_map",
           "quadrant_stats", "quadrant_stats_from_rows", "attention_quadrant_stats",
           "mask_recall"]
