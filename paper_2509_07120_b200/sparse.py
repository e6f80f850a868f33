"""Block-sparse global attention on the B200 (attention stage).

Drop-in for /root/reference/pkg/src/bsattn/sparse.py: ``SparseAttentionJob``
(:35-60), ``sparse_attention`` (:157-205), ``sparse_attention_stats``
(:208-236), ``flop_estimate`` (:253-259).  Special query rows attend every
key; patch query rows attend the special keys plus their selected key
blocks, merged with an online softmax; unselected blocks contribute nothing.

Device paths (chosen per call, both hand-written sm_100a CUDA):
  * tensor-core path (csrc/bsa_attn_tc.cu): bf16 inputs, head_dim 64,
    128x64 blocks -- TMA + tcgen05.mma + TMEM, persistent LPT schedule;
  * CUDA-core path (csrc/bsa_attn_simt.cu): fp32 math for fp32 inputs and
    every other geometry.
``panel_blocks`` and ``threads`` are accepted for API compatibility; the
kernel's own grouping (two key blocks per MMA tile) does not change results
beyond rounding, and the device result is identical for every host thread
count.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import NamedTuple

import numpy as np
import torch

from . import _native as N
from .dense import AttentionInputs
from .layout import TokenLayout
from .maskpred import BlockMask, MaskPolicy

DEFAULT_PANEL_BLOCKS = 32

_PATHS = {"auto": N.PATH_AUTO, "simt": N.PATH_SIMT, "tc": N.PATH_TC}


@dataclass(frozen=True)
class SparseAttentionJob:
    """Inputs, token layout and patch-patch block mask for one kernel run."""

    inputs: AttentionInputs
    layout: TokenLayout
    mask: BlockMask
    policy: MaskPolicy | None = None  # provenance echo only

    def __post_init__(self):
        n = self.inputs.tokens
        if n != self.layout.total_tokens:
            raise ValueError(
                f"inputs have {n} tokens but layout describes {self.layout.total_tokens}")
        if self.mask.geometry.patch_tokens != self.layout.patch_tokens:
            raise ValueError(
                f"mask geometry covers {self.mask.geometry.patch_tokens} patch tokens, "
                f"layout has {self.layout.patch_tokens}")
        if self.mask.heads != self.inputs.heads:
            raise ValueError(
                f"mask has {self.mask.heads} heads, inputs have {self.inputs.heads}")
        # host-built masks were checked for empty rows at construction;
        # device-built masks select >= 1 block per row by construction.


class FlopEstimate(NamedTuple):
    dense_flops: int
    sparse_flops: int
    theoretical_speedup: float


@dataclass
class HeadReport:
    head: int
    achieved_sparsity: float
    sparse_flops: int
    theoretical_speedup: float
    wall_ms: float


def attention_path(job: SparseAttentionJob, path: str = "auto") -> str:
    """Which device kernel ``sparse_attention`` uses for this job."""
    g = job.mask.geometry
    code = N.lib().bsa_sparse_attention_path(
        N.layout_desc(job.layout), job.inputs.head_dim, g.block_q, g.block_k,
        N.BSA_BF16 if job.inputs.q.dtype == torch.bfloat16 else N.BSA_F32, _PATHS[path])
    if code < 0:
        raise ValueError("tensor-core path needs bf16 or fp32 inputs, head_dim 64, block_q 128, block_k 64")
    return "tc" if code == N.PATH_TC else "simt"


def _flags(path: str, timing: bool, key_ranges: int, schedule: str = "lpt") -> int:
    if not 0 <= int(key_ranges) <= 255:
        raise ValueError(f"key_ranges must be in [0, 255], got {key_ranges}")
    if schedule not in ("lpt", "natural"):
        raise ValueError(f"schedule must be 'lpt' or 'natural', got {schedule!r}")
    return (_PATHS[path] | (N.FLAG_TIMING if timing else 0) | (int(key_ranges) << 8)
            | (N.FLAG_NATURAL_ORDER if schedule == "natural" else 0))


def _run(q, k, v, out, layout, mask: BlockMask, bits, counts, scale, inputs_permuted, shard,
         num_shards, path, ws=None, timing=False, key_ranges=0, schedule="lpt"):
    g = mask.geometry
    L = N.lib()
    lay = N.layout_desc(layout)
    in_code = N.BSA_BF16 if q.dtype == torch.bfloat16 else N.BSA_F32
    out_code = N.BSA_BF16 if out.dtype == torch.bfloat16 else N.BSA_F32
    flags = _flags(path, timing, key_ranges, schedule)
    need = L.bsa_sparse_attention_workspace(lay, q.shape[0], q.shape[2], g.block_q, g.block_k,
                                            in_code, int(inputs_permuted), flags)
    if ws is None or ws.numel() < need or ws.device != q.device:
        ws = N.workspace(need, q.device)
    with N.on_device(q.device):
        N.check(L.bsa_sparse_attention(
            N.tensor_desc(q), N.tensor_desc(k), N.tensor_desc(v), out.data_ptr(), out_code, lay,
            g.block_q, g.block_k, bits.data_ptr(), N.ptr(counts), np.float32(scale).item(),
            int(inputs_permuted), int(shard), int(num_shards), flags, ws.data_ptr(), ws.numel(),
            N.stream_ptr()), "sparse_attention")
    return ws


def _check_out(out: torch.Tensor, q: torch.Tensor, out_dtype) -> None:
    """The kernels write a contiguous (H, T, d) fp32/bf16 buffer on q's
    device through a raw pointer: anything else is refused up front."""
    if not isinstance(out, torch.Tensor):
        raise ValueError(f"out must be a torch tensor, got {type(out).__name__}")
    if tuple(out.shape) != tuple(q.shape):
        raise ValueError(f"out has shape {tuple(out.shape)}, expected {tuple(q.shape)}")
    if out.dtype not in (torch.float32, torch.bfloat16):
        raise ValueError(f"out dtype must be float32 or bfloat16, got {out.dtype}")
    if out_dtype is not None and out_dtype != out.dtype:
        raise ValueError(f"out_dtype {out_dtype} conflicts with out.dtype {out.dtype}")
    if out.device != q.device:
        raise ValueError(f"out is on {out.device}, inputs on {q.device}")
    if not out.is_contiguous():
        raise ValueError("out must be contiguous")


def kernel_times(max_n: int = 64, reset: bool = True) -> list[float]:
    """Device times (ms) of the most recent ``timing=True`` tensor-core
    kernel launches on this thread, oldest first (up to 64, no host sync
    needed between the launches); ``reset`` starts a new series."""
    buf = (ctypes.c_float * max(1, max_n))()
    n = N.lib().bsa_kernel_times(ctypes.cast(buf, ctypes.c_void_p), int(max_n), int(reset))
    if n < 0:
        raise RuntimeError("kernel_times: CUDA error reading the timing events")
    return [float(buf[i]) for i in range(n)]


def last_kernel_ms() -> float:
    """Device time of the last tensor-core attention kernel launched with
    ``timing=True`` on this thread (synchronises on it)."""
    return float(N.lib().bsa_last_kernel_ms())


def sparse_attention(job: SparseAttentionJob, *, panel_blocks: int = DEFAULT_PANEL_BLOCKS,
                     threads: int = 1, inputs_permuted: bool = False, out_dtype=None,
                     path: str = "auto", shard: int = 0, num_shards: int = 1, out=None,
                     workspace=None, timing: bool = False, key_ranges: int = 0,
                     schedule: str = "lpt"):
    """Run the block-sparse kernel; returns (heads, tokens, head_dim).

    Inputs arrive in interleaved source order and the result comes back in
    that order; with ``inputs_permuted=True`` both are [specials | patches].
    ``shard``/``num_shards`` compute only that shard's rows (every
    num_shards-th row of each head's LPT order; multi-GPU); other rows of
    ``out`` are left untouched.  ``key_ranges`` (tensor-core path): 0 picks
    the key-range split automatically (heads whose K/V outgrow L2 are cut
    into L2-sized key ranges, merged by log-sum-exp), n forces n ranges.
    ``schedule="natural"`` keeps each head's rows in index order instead of
    longest-first (to measure what the LPT order buys; same results).
    """
    del panel_blocks, threads
    inp = job.inputs
    q, k, v = inp.q, inp.k, inp.v
    if out is not None:
        _check_out(out, q, out_dtype)
    else:
        if out_dtype is None:
            out_dtype = q.dtype
        if out_dtype not in (torch.float32, torch.bfloat16):
            raise ValueError(f"out_dtype must be float32 or bfloat16, got {out_dtype}")
        alloc = torch.zeros if num_shards > 1 else torch.empty
        out = alloc(q.shape, dtype=out_dtype, device=q.device)
    bits = job.mask.device_bits(q.device)
    _run(q, k, v, out, job.layout, job.mask, bits, job.mask.device_counts(q.device), inp.scale,
         inputs_permuted, shard, num_shards, path, workspace, timing, key_ranges, schedule)
    if inp.numpy_io:
        return out.float().cpu().numpy()
    return out


def _flops_per_head(job: SparseAttentionJob):
    n = job.layout.total_tokens
    ns = job.layout.special_tokens
    npatch = job.layout.patch_tokens
    d = job.inputs.head_dim
    dense = 2 * n * n * d
    areas = job.mask.selected_area()
    sparse = [2 * d * (ns * n + npatch * ns + int(a)) for a in areas]
    return dense, sparse


def flop_estimate(job: SparseAttentionJob) -> FlopEstimate:
    """Multiply-accumulate counts of QK^T and PV, dense vs masked (the
    reference's naming: 'flops' counts MACs; sparse.py:239-259)."""
    per_dense, per_sparse = _flops_per_head(job)
    dense = per_dense * job.inputs.heads
    sparse = sum(per_sparse)
    return FlopEstimate(dense, sparse, dense / sparse)


def sparse_attention_stats(job: SparseAttentionJob, *,
                           panel_blocks: int = DEFAULT_PANEL_BLOCKS, path: str = "auto"):
    """sparse_attention plus per-head sparsity, MAC counts and device time
    (CUDA events around one launch per head)."""
    del panel_blocks
    inp = job.inputs
    q, k, v = inp.q, inp.k, inp.v
    g = job.mask.geometry
    out = torch.empty(q.shape, dtype=q.dtype, device=q.device)
    bits = job.mask.device_bits(q.device)
    counts = job.mask.device_counts(q.device)
    sparsity = job.mask.achieved_sparsity()
    per_dense, per_sparse = _flops_per_head(job)
    reports = []
    rows = g.nq_blocks
    for h in range(inp.heads):
        sub = BlockMask._from_device(bits[h * rows:(h + 1) * rows], None, 1, g)
        c = counts[h * rows:(h + 1) * rows] if counts is not None else None
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        stream = torch.cuda.current_stream(q.device)
        e0.record(stream)
        _run(q[h:h + 1], k[h:h + 1], v[h:h + 1], out[h:h + 1], job.layout, sub, sub._bits, c,
             inp.scale, False, 0, 1, path)
        e1.record(stream)
        e1.synchronize()
        reports.append(HeadReport(
            head=h,
            achieved_sparsity=float(sparsity[h]),
            sparse_flops=int(per_sparse[h]),
            theoretical_speedup=per_dense / per_sparse[h],
            wall_ms=float(e0.elapsed_time(e1)),
        ))
    res = out.float().cpu().numpy() if inp.numpy_io else out
    return res, reports
