"""Training-free block-mask prediction on the B200 (scoring stage).

Drop-in for /root/reference/pkg/src/bsattn/maskpred.py: same names, argument
meaning, ValueError behaviour and .bsm format.  The arithmetic runs in the
sm_100a kernels of libbsa.so (csrc/bsa_score.cu) and reproduces the
reference's fp32 results bit for bit: pooled block means, pooled
probabilities and the selected-block masks.

Arrays may be numpy (results come back as numpy, like the reference) or
torch CUDA tensors (results stay on the device).  A BlockMask keeps its
bitsets on the device in .bsm row layout and only materialises the boolean
``blocks`` array when asked.
"""

from __future__ import annotations

import struct
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from .layout import BlockGeometry, TokenLayout

MASK_MAGIC = b"BSMK"
_MASK_HEADER_FMT = "<4sIII"
_MASK_HEADER_SIZE = struct.calcsize(_MASK_HEADER_FMT)


# ---------------------------------------------------------------------------
# input plumbing
# ---------------------------------------------------------------------------
def _to_device(x, name: str, allow_bf16: bool = True, validate: bool = True):
    """-> (contiguous-last-dim CUDA tensor, came_from_numpy).

    validate: reject NaN/inf like the reference's as_f32 (tensorio.py:47-59)
    for every input, device tensors included (one min/max reduction and one
    sync per tensor; callers that validated already pass False)."""
    dev = N.require_cuda()
    if isinstance(x, torch.Tensor):
        t = x
        if t.dim() == 0:
            raise ValueError(f"{name} must have at least one dimension")
        if min(t.shape) < 1:
            raise ValueError(f"{name} has a zero-sized dimension: {tuple(t.shape)}")
        if t.dtype not in ((torch.float32, torch.bfloat16) if allow_bf16 else (torch.float32,)):
            t = t.float()
        if t.device.type != "cuda":
            if validate and not torch.isfinite(t).all():
                raise ValueError(f"{name} contains non-finite values")
            t = t.to(dev)
        elif validate and not N.all_finite(t):
            raise ValueError(f"{name} contains non-finite values")
        if t.stride(-1) != 1:
            t = t.contiguous()
        return t, False
    a = np.asarray(x, dtype=np.float32)
    if a.ndim == 0:
        raise ValueError(f"{name} must have at least one dimension")
    if min(a.shape) < 1:
        raise ValueError(f"{name} has a zero-sized dimension: {a.shape}")
    if validate and not np.isfinite(a).all():
        raise ValueError(f"{name} contains non-finite values")
    return torch.from_numpy(np.ascontiguousarray(a)).to(dev), True


def _out(t: torch.Tensor, numpy_out: bool):
    return t.cpu().numpy() if numpy_out else t


# ---------------------------------------------------------------------------
# policy / mask types
# ---------------------------------------------------------------------------
@dataclass(frozen=True)
class MaskPolicy:
    """CDF threshold tau, sparse ratio rho, block geometry (maskpred.py:38-57)."""

    tau: float
    rho: float
    geometry: BlockGeometry

    def __post_init__(self):
        if not 0.0 <= self.tau <= 1.0:
            raise ValueError(f"tau must be in [0, 1], got {self.tau}")
        if not 0.0 <= self.rho <= 1.0:
            raise ValueError(f"rho must be in [0, 1], got {self.rho}")

    @property
    def min_blocks(self) -> int:
        """floor(nk * (1 - rho)) clamped to [1, nk]; the +1e-9 keeps exact
        products such as 100 * (1 - 0.9) from flooring low."""
        nk = self.geometry.nk_blocks
        return min(nk, max(1, int(nk * (1.0 - self.rho) + 1e-9)))


class BlockMask:
    """Per-head key-block selection for every query-block row.

    Construct from a boolean (heads, nq, nk) array like the reference
    (maskpred.py:60-101); device-produced masks carry their .bsm bitsets and
    per-row counts on the GPU and decode ``blocks`` lazily.
    """

    def __init__(self, blocks, geometry: BlockGeometry):
        if isinstance(blocks, torch.Tensor):
            blocks = blocks.detach().cpu().numpy()
        b = np.ascontiguousarray(blocks, dtype=bool)
        if b.ndim != 3:
            raise ValueError(f"blocks must be (heads, nq, nk), got {b.shape}")
        if b.shape[1] != geometry.nq_blocks or b.shape[2] != geometry.nk_blocks:
            raise ValueError(
                f"mask shape {b.shape[1:]} inconsistent with geometry "
                f"({geometry.nq_blocks}, {geometry.nk_blocks})")
        if not b.any(axis=2).all():
            raise ValueError("every query-block row must select at least one key block")
        self.geometry = geometry
        self._heads = b.shape[0]
        self._blocks = b
        self._bits = None
        self._counts = None

    @classmethod
    def _from_device(cls, bits: torch.Tensor, counts: torch.Tensor, heads: int,
                     geometry: BlockGeometry) -> "BlockMask":
        m = cls.__new__(cls)
        m.geometry = geometry
        m._heads = heads
        m._blocks = None
        m._bits = bits
        m._counts = counts
        return m

    # -- reference surface -------------------------------------------------
    @property
    def heads(self) -> int:
        return self._heads

    @property
    def blocks(self) -> np.ndarray:
        if self._blocks is None:
            g = self.geometry
            packed = self._bits.cpu().numpy()
            bits = np.unpackbits(packed, axis=1, bitorder="little")[:, : g.nk_blocks]
            self._blocks = bits.astype(bool).reshape(self._heads, g.nq_blocks, g.nk_blocks)
        return self._blocks

    def selected_area(self) -> np.ndarray:
        """Selected patch-patch entries per head, int64 (maskpred.py:97-101)."""
        g = self.geometry
        bits = self.device_bits()
        area = torch.empty(self._heads, dtype=torch.int64, device=bits.device)
        with N.on_device(bits.device):
            N.check(N.lib().bsa_mask_selected_area(bits.data_ptr(), self._heads, g.patch_tokens,
                                                   g.block_q, g.block_k, area.data_ptr(),
                                                   N.stream_ptr()), "selected_area")
        return area.cpu().numpy()

    def achieved_sparsity(self) -> np.ndarray:
        """Fraction of patch-patch entries not selected, per head (float64,
        ragged tails weighted by their true size; maskpred.py:85-95)."""
        total = float(self.geometry.patch_tokens) ** 2
        return 1.0 - self.selected_area().astype(np.float64) / total

    # -- device views --------------------------------------------------------
    def device_bits(self, device=None) -> torch.Tensor:
        """(heads*nq, ceil(nk/8)) uint8 on the GPU, .bsm row layout.  With
        `device`, the bits are moved there (and cached there) if they live
        on another GPU."""
        if self._bits is None:
            dev = device or N.require_cuda()
            g = self.geometry
            packed = np.packbits(self._blocks.reshape(-1, g.nk_blocks), axis=1, bitorder="little")
            self._bits = torch.from_numpy(np.ascontiguousarray(packed)).to(dev)
        elif device is not None and self._bits.device != torch.device(device):
            self._bits = self._bits.to(device)
            if self._counts is not None:
                self._counts = self._counts.to(device)
        return self._bits

    def device_counts(self, device=None) -> torch.Tensor | None:
        if device is not None and self._counts is not None and \
                self._counts.device != torch.device(device):
            self._counts = self._counts.to(device)
        return self._counts

    def csr(self):
        """(row_ptr int32[H*nq+1], col_idx int32[nnz]) on the device."""
        g = self.geometry
        bits = self.device_bits()
        rows = self._heads * g.nq_blocks
        L = N.lib()
        ws = N.workspace(L.bsa_mask_to_csr_workspace(self._heads, g.nq_blocks), bits.device)
        row_ptr = torch.empty(rows + 1, dtype=torch.int32, device=bits.device)
        nnz = int(np.unpackbits(bits.cpu().numpy(), axis=1, bitorder="little")[:, : g.nk_blocks].sum())
        col_idx = torch.empty(max(nnz, 1), dtype=torch.int32, device=bits.device)
        with N.on_device(bits.device):
            N.check(L.bsa_mask_to_csr(bits.data_ptr(), self._heads, g.nq_blocks, g.nk_blocks,
                                      row_ptr.data_ptr(), col_idx.data_ptr(), ws.data_ptr(),
                                      ws.numel(), N.stream_ptr()), "mask_to_csr")
        return row_ptr, col_idx[:nnz]


# ---------------------------------------------------------------------------
# operators
# ---------------------------------------------------------------------------
def block_pool(x, block: int, *, validate: bool = True):
    """Average-pool (heads, tokens, dim) over token blocks (maskpred.py:104-120)."""
    t, was_np = _to_device(x, "x", validate=validate)
    if t.dim() != 3:
        raise ValueError(f"block_pool expects (heads, tokens, dim), got {tuple(t.shape)}")
    if block < 1:
        raise ValueError(f"block size must be >= 1, got {block}")
    h, n, d = t.shape
    out = torch.empty((h, -(-n // block), d), dtype=torch.float32, device=t.device)
    with N.on_device(t.device):
        N.check(N.lib().bsa_block_pool(N.tensor_desc(t), None, int(block), out.data_ptr(),
                                       N.stream_ptr()), "block_pool")
    return _out(out, was_np)


def pooled_scores(q_pooled, k_pooled, head_dim: int, *, validate: bool = True):
    """Softmaxed pooled similarity (heads, nq, nk) (maskpred.py:123-139)."""
    qp, was_np = _to_device(q_pooled, "q_pooled", allow_bf16=False, validate=validate)
    kp, _ = _to_device(k_pooled, "k_pooled", allow_bf16=False, validate=validate)
    if kp.device != qp.device:
        raise ValueError(f"q_pooled on {qp.device} but k_pooled on {kp.device}")
    if qp.dim() != 3 or kp.dim() != 3:
        raise ValueError(f"pooled tensors must be 3-D, got {tuple(qp.shape)} and {tuple(kp.shape)}")
    if qp.shape[0] != kp.shape[0] or qp.shape[2] != kp.shape[2]:
        raise ValueError(f"pooled shapes incompatible: {tuple(qp.shape)} vs {tuple(kp.shape)}")
    qp, kp = qp.contiguous(), kp.contiguous()
    h, nq, d = qp.shape
    nk = kp.shape[1]
    scale = np.float32(1.0 / float(np.sqrt(head_dim)))
    out = torch.empty((h, nq, nk), dtype=torch.float32, device=qp.device)
    L = N.lib()
    ws = N.workspace(L.bsa_pooled_scores_workspace(h, nq, nk), qp.device)
    with N.on_device(qp.device):
        N.check(L.bsa_pooled_scores(qp.data_ptr(), kp.data_ptr(), h, nq, nk, d, float(scale),
                                    out.data_ptr(), ws.data_ptr(), ws.numel(), N.stream_ptr()),
                "pooled_scores")
    return _out(out, was_np)


def select_blocks(scores, policy: MaskPolicy, *, validate: bool = True) -> BlockMask:
    """Per (head, q-block) row: rank blocks by probability (ties -> lower
    index), shortest prefix reaching tau, extended to the rho floor
    (maskpred.py:142-174)."""
    s, _ = _to_device(scores, "scores", allow_bf16=False, validate=validate)
    if s.dim() != 3:
        raise ValueError(f"scores must be (heads, nq, nk), got {tuple(s.shape)}")
    g = policy.geometry
    if s.shape[1] != g.nq_blocks or s.shape[2] != g.nk_blocks:
        raise ValueError(
            f"scores shape {tuple(s.shape[1:])} inconsistent with geometry "
            f"({g.nq_blocks}, {g.nk_blocks})")
    s = s.contiguous()
    h, nq, nk = s.shape
    L = N.lib()
    bits = torch.empty((h * nq, -(-nk // 8)), dtype=torch.uint8, device=s.device)
    counts = torch.empty(h * nq, dtype=torch.int32, device=s.device)
    ws = N.workspace(L.bsa_select_workspace(h, nq, nk), s.device)
    with N.on_device(s.device):
        N.check(L.bsa_select_blocks(s.data_ptr(), h, nq, nk, float(policy.tau),
                                    policy.min_blocks, bits.data_ptr(), counts.data_ptr(),
                                    ws.data_ptr(), ws.numel(), N.stream_ptr()), "select_blocks")
    return BlockMask._from_device(bits, counts, h, g)


def predict_mask(q_patches, k_patches, policy: MaskPolicy, *, layout: TokenLayout | None = None,
                 return_probs: bool = False, validate: bool = True):
    """Pool, score and select in one device pass (maskpred.py:177-194).

    Inputs are (heads, patch_tokens, head_dim) patch-only tensors, exactly as
    the reference.  Extension: with ``layout=`` they may instead be the full
    interleaved sequences; the patch gather is then folded into the kernels'
    addressing (no copy).  ``validate=False`` skips the non-finite scan of
    the inputs (as_f32, tensorio.py:47-59) for callers that already did it.
    """
    q, _ = _to_device(q_patches, "q_patches", validate=validate)
    k, _ = _to_device(k_patches, "k_patches", validate=validate)
    if k.device != q.device:
        raise ValueError(f"q on {q.device} but k on {k.device}")
    g = policy.geometry
    expect = layout.total_tokens if layout is not None else g.patch_tokens
    if layout is not None and layout.patch_tokens != g.patch_tokens:
        raise ValueError(f"layout has {layout.patch_tokens} patch tokens, geometry {g.patch_tokens}")
    if q.dim() != 3 or k.dim() != 3:
        raise ValueError("q/k must be (heads, tokens, head_dim)")
    if q.shape[1] != expect or k.shape[1] != expect:
        raise ValueError(f"expected {expect} patch tokens, got q={q.shape[1]}, k={k.shape[1]}")
    if q.shape != k.shape:
        raise ValueError(f"q/k shapes differ: {tuple(q.shape)} vs {tuple(k.shape)}")
    if q.dtype != k.dtype:
        # promote like the reference (as_f32 makes both fp32, tensorio.py:47-59)
        q, k = q.float(), k.float()
    h, _, d = q.shape
    L = N.lib()
    nq, nk = g.nq_blocks, g.nk_blocks
    bits = torch.empty((h * nq, -(-nk // 8)), dtype=torch.uint8, device=q.device)
    counts = torch.empty(h * nq, dtype=torch.int32, device=q.device)
    probs = torch.empty((h, nq, nk), dtype=torch.float32, device=q.device) if return_probs else None
    ws = N.workspace(L.bsa_predict_mask_workspace(h, g.patch_tokens, d, g.block_q, g.block_k),
                     q.device)
    scale = np.float32(1.0 / float(np.sqrt(d)))
    lay = N.layout_desc(layout) if layout is not None else None
    with N.on_device(q.device):
        N.check(L.bsa_predict_mask(N.tensor_desc(q), N.tensor_desc(k), lay, g.block_q, g.block_k,
                                   float(scale), float(policy.tau), policy.min_blocks,
                                   bits.data_ptr(), counts.data_ptr(), N.ptr(probs),
                                   ws.data_ptr(), ws.numel(), N.stream_ptr()), "predict_mask")
    mask = BlockMask._from_device(bits, counts, h, g)
    if return_probs:
        return mask, probs
    return mask


def predict_mask_pooled(q_pooled, k_pooled, policy: MaskPolicy, *, return_probs: bool = False,
                        validate: bool = True):
    """predict_mask from block means already pooled (maskpred.py:177-194
    minus its two block_pool calls): (heads, nq, d) / (heads, nk, d) fp32,
    e.g. the QKV-projection epilogue's (qkv.qkv_projection).  Same mask and
    probabilities as predict_mask on the tensors they were pooled from."""
    qp, _ = _to_device(q_pooled, "q_pooled", allow_bf16=False, validate=validate)
    kp, _ = _to_device(k_pooled, "k_pooled", allow_bf16=False, validate=validate)
    if kp.device != qp.device:
        raise ValueError(f"q_pooled on {qp.device} but k_pooled on {kp.device}")
    if qp.dim() != 3 or kp.dim() != 3:
        raise ValueError(f"pooled tensors must be 3-D, got {tuple(qp.shape)} and {tuple(kp.shape)}")
    g = policy.geometry
    if qp.shape[1] != g.nq_blocks or kp.shape[1] != g.nk_blocks:
        raise ValueError(f"pooled shapes {tuple(qp.shape)} / {tuple(kp.shape)} inconsistent with "
                         f"geometry ({g.nq_blocks}, {g.nk_blocks})")
    if qp.shape[0] != kp.shape[0] or qp.shape[2] != kp.shape[2]:
        raise ValueError(f"pooled shapes incompatible: {tuple(qp.shape)} vs {tuple(kp.shape)}")
    qp, kp = qp.contiguous(), kp.contiguous()
    h, nq, d = qp.shape
    nk = kp.shape[1]
    L = N.lib()
    bits = torch.empty((h * nq, -(-nk // 8)), dtype=torch.uint8, device=qp.device)
    counts = torch.empty(h * nq, dtype=torch.int32, device=qp.device)
    probs = torch.empty((h, nq, nk), dtype=torch.float32, device=qp.device) if return_probs else None
    ws = N.workspace(L.bsa_predict_mask_pooled_workspace(h, nq, nk, d), qp.device)
    scale = np.float32(1.0 / float(np.sqrt(d)))
    with N.on_device(qp.device):
        N.check(L.bsa_predict_mask_pooled(qp.data_ptr(), kp.data_ptr(), h, nq, nk, d, float(scale),
                                          float(policy.tau), policy.min_blocks, bits.data_ptr(),
                                          counts.data_ptr(), N.ptr(probs), ws.data_ptr(),
                                          ws.numel(), N.stream_ptr()), "predict_mask_pooled")
    mask = BlockMask._from_device(bits, counts, h, g)
    if return_probs:
        return mask, probs
    return mask


def full_mask(geometry: BlockGeometry, heads: int) -> BlockMask:
    """All-selected mask (sparsity zero)."""
    return BlockMask(np.ones((heads, geometry.nq_blocks, geometry.nk_blocks), dtype=bool), geometry)


def write_mask(path, mask: BlockMask) -> None:
    """.bsm: magic, heads, nq, nk (u32 LE), then LSB-first row bitsets."""
    g = mask.geometry
    if mask._bits is not None:
        payload = mask._bits.cpu().numpy().tobytes()
    else:
        payload = np.packbits(mask._blocks.reshape(-1, g.nk_blocks), axis=1,
                              bitorder="little").tobytes()
    with open(path, "wb") as f:
        f.write(struct.pack(_MASK_HEADER_FMT, MASK_MAGIC, mask.heads, g.nq_blocks, g.nk_blocks))
        f.write(payload)


def read_mask(path, geometry: BlockGeometry) -> BlockMask:
    with open(path, "rb") as f:
        raw = f.read()
    if len(raw) < _MASK_HEADER_SIZE:
        raise ValueError(f"mask file too short for header: {len(raw)} bytes")
    magic, h, nq, nk = struct.unpack_from(_MASK_HEADER_FMT, raw, 0)
    if magic != MASK_MAGIC:
        raise ValueError(f"bad mask magic {magic!r}, expected {MASK_MAGIC!r}")
    if min(h, nq, nk) < 1:
        raise ValueError(f"invalid mask header dims ({h}, {nq}, {nk})")
    row_bytes = -(-nk // 8)
    expected = _MASK_HEADER_SIZE + h * nq * row_bytes
    if len(raw) != expected:
        raise ValueError(f"mask file size {len(raw)} != expected {expected}")
    packed = np.frombuffer(raw, dtype=np.uint8, offset=_MASK_HEADER_SIZE).reshape(h * nq, row_bytes)
    bits = np.unpackbits(packed, axis=1, bitorder="little")[:, :nk]
    return BlockMask(bits.astype(bool).reshape(h, nq, nk), geometry)
