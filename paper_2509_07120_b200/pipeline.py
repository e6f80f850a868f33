"""One block-sparse global-attention layer from HOST memory, with the PCIe
copies overlapped with the kernels.

Attention heads are independent all the way through the path: pooling,
scoring, selection (maskpred.py:104-174 work per head) and the
block-sparse kernel (sparse.py:134-154 ``_run_head``). The layer therefore
runs as a pipeline over chunks of heads on three CUDA streams:

    copy-in stream   H2D  Q/K/V of chunk c+1   (pinned host -> HBM)
    compute stream   predict_mask + sparse_attention of chunk c
    copy-out stream  D2H  output of chunk c-1  (HBM -> pinned host)

The layer costs about max(compute, copies) plus one chunk of ramp, instead
of copy-in + compute + copy-out. This is the public entry point a caller
with host-resident activations uses, and bench.py's ``e2e`` measurement.
"""

from __future__ import annotations

import torch

from . import _native as N
from .dense import AttentionInputs
from .layout import TokenLayout
from .maskpred import BlockMask, MaskPolicy, predict_mask
from .sparse import SparseAttentionJob, sparse_attention


def ramp_chunks(heads: int, peak: int = 4) -> list[int]:
    """Chunk sizes 1, 3, peak, ..., peak, 3, 1: one-head chunks at both ends
    keep the uncovered first H2D and last D2H short; larger middle chunks
    keep the kernels efficient (measured best at H=16: 1,3,4,4,3,1)."""
    if heads <= 2:
        return [1] * heads
    ends = [1, 3] if heads >= 8 else [1]
    mid = heads - 2 * sum(ends)
    n = -(-mid // peak)  # middle chunks, as even as possible
    sizes = [mid // n + (1 if i < mid % n else 0) for i in range(n)] if mid else []
    return ends + sizes + ends[::-1]


class HostLayerPipeline:
    """Reusable device buffers and streams for repeated layers of one shape."""

    def __init__(self, heads: int, tokens: int, head_dim: int, dtype=torch.bfloat16,
                 chunk_heads="auto", device=None, partitioned_copies: bool = True):
        """chunk_heads: heads per pipeline chunk, the list of chunk sizes
        (summing to `heads`), or "auto" (ramp_chunks). Small first and last
        chunks shorten the ramp: the first H2D and the last D2H are the only
        uncovered copies.

        partitioned_copies: the copy engines reorder tokens on the way in
        (interleaved host rows -> partitioned device rows, two strided copies
        per head: bsa_copy_tokens) and back on the way out, so the kernels
        read Q/K/V in place (no pack pass) and score contiguous patch rows."""
        if isinstance(chunk_heads, str):
            if chunk_heads != "auto":
                raise ValueError(f"chunk_heads must be an int, a list or 'auto', got {chunk_heads!r}")
            sizes = ramp_chunks(heads)
        elif isinstance(chunk_heads, int):
            if chunk_heads < 1:
                raise ValueError(f"chunk_heads must be >= 1, got {chunk_heads}")
            c = min(chunk_heads, heads)
            sizes = [min(c, heads - h0) for h0 in range(0, heads, c)]
        else:
            sizes = [int(x) for x in chunk_heads]
            if any(x < 1 for x in sizes) or sum(sizes) != heads:
                raise ValueError(f"chunk sizes {sizes} must be >= 1 and sum to {heads}")
        self.device = torch.device(device or "cuda")
        self.shape = (heads, tokens, head_dim)
        self.dtype = dtype
        self.chunks = []
        h0 = 0
        for x in sizes:
            self.chunks.append((h0, h0 + x))
            h0 += x
        self.bufs = [torch.empty(self.shape, dtype=dtype, device=self.device) for _ in range(3)]
        self.obuf = torch.empty(self.shape, dtype=dtype, device=self.device)
        self.partitioned = bool(partitioned_copies)
        self.s_in = torch.cuda.Stream(self.device)
        self.s_out = torch.cuda.Stream(self.device)

    def run(self, q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, layout: TokenLayout,
            policy: MaskPolicy, out: torch.Tensor | None = None, return_masks: bool = False,
            validate: bool = True):
        """q, k, v: host (ideally pinned) (H, T, d) tensors in interleaved
        token order. Returns the host output (and the per-chunk masks).
        The call is synchronous: the output is complete on return.

        validate: reject non-finite inputs like the reference's as_f32
        (tensorio.py:47-59). The scan runs on the device copy of each chunk,
        asynchronously, and is checked once at the end (a host scan of the
        pinned buffers, or a sync per chunk, would stall the pipeline)."""
        for name, t in (("q", q), ("k", k), ("v", v)):
            if tuple(t.shape) != self.shape or t.dtype != self.dtype:
                raise ValueError(f"{name} must be {self.shape} {self.dtype}, got "
                                 f"{tuple(t.shape)} {t.dtype}")
            if t.device.type != "cpu":
                raise ValueError(f"{name} must be a host tensor (use sparse_attention for "
                                 f"device-resident inputs)")
        if out is None:
            out = torch.empty(self.shape, dtype=self.dtype, pin_memory=True)
        dq, dk, dv = self.bufs
        comp = torch.cuda.current_stream(self.device)
        masks = []
        bad = torch.zeros(1, dtype=torch.int32, device=self.device) if validate else None
        done_in, done_comp = [], []
        chunks = self.chunks
        # the copy-in stream must not overwrite buffers a previous call still reads
        self.s_in.wait_stream(comp)
        part = self.partitioned
        if part:
            for name, t in (("q", q), ("k", k), ("v", v)):
                if not t.is_contiguous():
                    raise ValueError(f"{name} must be contiguous")
            if layout.total_tokens != self.shape[1]:
                raise ValueError(f"layout has {layout.total_tokens} tokens, buffers {self.shape[1]}")
            lay_d = N.layout_desc(layout)
            row = self.shape[2] * q.element_size()
            Ts = layout.special_tokens

        def copy_in(dst, src, a, b):
            if part:
                N.check(N.lib().bsa_copy_tokens(dst[a:b].data_ptr(), src[a:b].data_ptr(), lay_d,
                                                b - a, row, 1, self.s_in.cuda_stream), "copy_tokens")
            else:
                dst[a:b].copy_(src[a:b], non_blocking=True)

        for a, b in chunks:
            with torch.cuda.stream(self.s_in):
                # Q and K first: scoring can start while V is still in flight
                copy_in(dq, q, a, b)
                copy_in(dk, k, a, b)
                ev_qk = torch.cuda.Event()
                ev_qk.record(self.s_in)
                copy_in(dv, v, a, b)
                ev_v = torch.cuda.Event()
                ev_v.record(self.s_in)
                done_in.append((ev_qk, ev_v))
        for (a, b), (ev_qk, ev_v) in zip(chunks, done_in):
            comp.wait_event(ev_qk)
            if part:  # patch rows are contiguous after the specials
                mask = predict_mask(dq[a:b, Ts:], dk[a:b, Ts:], policy, validate=False)
            else:
                mask = predict_mask(dq[a:b], dk[a:b], policy, layout=layout, validate=False)
            comp.wait_event(ev_v)
            if validate:  # device scan into one flag, read once at the end
                for x in (dq, dk, dv):
                    N.finite_scan(x[a:b], bad)
            job = SparseAttentionJob(AttentionInputs(dq[a:b], dk[a:b], dv[a:b], validate=False),
                                     layout, mask)
            sparse_attention(job, out=self.obuf[a:b], inputs_permuted=part)
            ev = torch.cuda.Event()
            ev.record(comp)
            done_comp.append(ev)
            if return_masks:
                masks.append(mask)
            with torch.cuda.stream(self.s_out):
                self.s_out.wait_event(ev)
                if part:  # back to the caller's interleaved token order
                    N.check(N.lib().bsa_copy_tokens(out[a:b].data_ptr(), self.obuf[a:b].data_ptr(),
                                                    lay_d, b - a, row, 0, self.s_out.cuda_stream),
                            "copy_tokens")
                else:
                    out[a:b].copy_(self.obuf[a:b], non_blocking=True)
        comp.wait_stream(self.s_out)
        torch.cuda.current_stream(self.device).synchronize()
        if validate and int(bad.item()) != 0:
            raise ValueError("q/k/v contain non-finite values")
        return (out, masks) if return_masks else out


def attend_from_host(q, k, v, layout: TokenLayout, policy: MaskPolicy, *, chunk_heads="auto",
                     out=None):
    """One-shot convenience wrapper around HostLayerPipeline."""
    p = HostLayerPipeline(q.shape[0], q.shape[1], q.shape[2], q.dtype, chunk_heads)
    return p.run(q, k, v, layout, policy, out)


__all__ = ["HostLayerPipeline", "attend_from_host", "ramp_chunks", "BlockMask"]
