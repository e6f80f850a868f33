"""CPU oracle for the block-sparse global-attention hot path.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py`` (its ``cpu_baseline`` leg and ``--impl reference``) may import
this package, and only as the checker / the timed CPU baseline.  The product
package ``paper_2509_07120_b200`` never imports it and has no CPU path.

Two parts:

* ``liboracle.so`` (``oracle/bsa_oracle.c``): the scoring stage restated in C
  with numpy/OpenBLAS's exact fp32 operation order, so block masks can be
  compared bit-for-bit.  Reference: maskpred.py:104-194, tensorio.py:73-87.
* numpy restatements of the attention stage (sparse.py:78-205, dense.py:58-76):
  ``sparse_attention_port`` streams the special strip and the selected key
  blocks with the reference's online-softmax update in fp32 (this is also the
  timed CPU baseline), and ``masked_attention_f64`` is an exact float64
  softmax over the allowed keys of chosen rows (the tight checker).

Pinning: ``tests/golden/make_golden.py`` ran the reference package
(/root/reference/pkg/src/bsattn) in the build container and committed its
outputs under ``tests/golden/``; ``tests/test_cpu_oracle_host.py`` checks this
oracle against those fixtures on every run.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from concurrent.futures import ThreadPoolExecutor

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None


def build() -> str:
    """Compile liboracle.so with the committed Makefile (gcc)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        src = os.path.join(_HERE, "bsa_oracle.c")
        if not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        i64, f32, f64 = ctypes.c_int64, ctypes.c_float, ctypes.c_double
        vp = ctypes.c_void_p
        L.oracle_np_expf.argtypes = [f32]
        L.oracle_np_expf.restype = f32
        L.oracle_pairwise_sum.argtypes = [vp, i64]
        L.oracle_pairwise_sum.restype = f32
        L.oracle_block_pool.argtypes = [vp, i64, i64, i64, i64, vp]
        L.oracle_pooled_scores.argtypes = [vp, vp, i64, i64, i64, i64, f32, vp]
        L.oracle_select_blocks.argtypes = [vp, i64, i64, i64, f64, i64, vp, vp]
        L.oracle_predict_mask.argtypes = [vp, vp, i64, i64, i64, i64, i64, f32, f64, i64,
                                          vp, vp, vp]
        L.oracle_num_threads.restype = ctypes.c_int
        _lib = L
    return _lib


def _f32c(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float32)


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _check(rc: int, what: str):
    if rc != 0:
        raise RuntimeError(f"oracle {what} failed with code {rc}")


def host_threads() -> int:
    return int(lib().oracle_num_threads())


# --------------------------------------------------------------------------
# scoring stage (bit-exact restatement)
# --------------------------------------------------------------------------
def head_scale(head_dim: int) -> float:
    """1/sqrt(d) in float64, as AttentionInputs.scale (dense.py:55)."""
    return 1.0 / float(np.sqrt(head_dim))


def min_blocks(nk: int, rho: float) -> int:
    """MaskPolicy.min_blocks (maskpred.py:52-57), same float64 expression."""
    return min(nk, max(1, int(nk * (1.0 - rho) + 1e-9)))


def np_expf(x: np.ndarray) -> np.ndarray:
    L = lib()
    flat = _f32c(x).ravel()
    return np.array([L.oracle_np_expf(float(v)) for v in flat], dtype=np.float32).reshape(np.shape(x))


def block_pool(x, block: int) -> np.ndarray:
    x = _f32c(x)
    h, n, d = x.shape
    nb = -(-n // block)
    out = np.empty((h, nb, d), dtype=np.float32)
    _check(lib().oracle_block_pool(_ptr(x), h, n, d, block, _ptr(out)), "block_pool")
    return out


def pooled_scores(qp, kp, head_dim: int) -> np.ndarray:
    qp, kp = _f32c(qp), _f32c(kp)
    h, nq, d = qp.shape
    nk = kp.shape[1]
    out = np.empty((h, nq, nk), dtype=np.float32)
    scale = np.float32(head_scale(head_dim))
    _check(lib().oracle_pooled_scores(_ptr(qp), _ptr(kp), h, nq, nk, d, float(scale), _ptr(out)),
           "pooled_scores")
    return out


def select_blocks(probs, tau: float, k_floor: int):
    """Returns (mask bool (H,nq,nk), per-row selected counts int32 (H,nq))."""
    p = _f32c(probs)
    h, nq, nk = p.shape
    mask = np.empty((h, nq, nk), dtype=np.uint8)
    counts = np.empty((h, nq), dtype=np.int32)
    _check(lib().oracle_select_blocks(_ptr(p), h, nq, nk, float(tau), int(k_floor), _ptr(mask),
                                      _ptr(counts)), "select_blocks")
    return mask.astype(bool), counts


def predict_mask(q_patches, k_patches, block_q: int, block_k: int, tau: float, rho: float,
                 return_probs: bool = False):
    q, k = _f32c(q_patches), _f32c(k_patches)
    h, tp, d = q.shape
    nq, nk = -(-tp // block_q), -(-tp // block_k)
    mask = np.empty((h, nq, nk), dtype=np.uint8)
    counts = np.empty((h, nq), dtype=np.int32)
    probs = np.empty((h, nq, nk), dtype=np.float32) if return_probs else None
    scale = np.float32(head_scale(d))
    _check(lib().oracle_predict_mask(_ptr(q), _ptr(k), h, tp, d, block_q, block_k, float(scale),
                                     float(tau), min_blocks(nk, rho), _ptr(mask), _ptr(counts),
                                     _ptr(probs) if probs is not None else None), "predict_mask")
    if return_probs:
        return mask.astype(bool), counts, probs
    return mask.astype(bool), counts


def pack_bits(mask: np.ndarray) -> np.ndarray:
    """(H,nq,nk) bool -> (H*nq, ceil(nk/8)) uint8, LSB-first (.bsm rows, maskpred.py:17-19)."""
    h, nq, nk = mask.shape
    return np.packbits(mask.reshape(h * nq, nk), axis=1, bitorder="little")


# --------------------------------------------------------------------------
# token layout (layout.py:113-143)
# --------------------------------------------------------------------------
def partition_perm(frames: int, patches: int, specials: int, specials_first: bool = True):
    """Gather permutation source order -> [all specials | all patches] and its inverse."""
    per = patches + specials
    base = np.arange(frames, dtype=np.int64)[:, None] * per
    if specials_first:
        spec = base + np.arange(specials, dtype=np.int64)
        pat = base + specials + np.arange(patches, dtype=np.int64)
    else:
        pat = base + np.arange(patches, dtype=np.int64)
        spec = base + patches + np.arange(specials, dtype=np.int64)
    perm = np.concatenate([spec.ravel(), pat.ravel()])
    inv = np.empty_like(perm)
    inv[perm] = np.arange(perm.size, dtype=np.int64)
    return perm, inv


def patch_indices(frames: int, patches: int, specials: int, specials_first: bool = True):
    perm, _ = partition_perm(frames, patches, specials, specials_first)
    return perm[frames * specials:]


# --------------------------------------------------------------------------
# attention stage
# --------------------------------------------------------------------------
def _row_keys(mask_row: np.ndarray, n_spec: int, tp: int, block_k: int) -> np.ndarray:
    """Partitioned-order key indices one patch q-block may see: the special
    strip, then each selected key block ascending (sparse.py:101-119)."""
    blocks = np.flatnonzero(mask_row)
    if blocks.size == 0:
        raise ValueError("patch row with empty key-block selection reached the kernel")
    pieces = [np.arange(n_spec, dtype=np.int64)]
    for b in blocks:
        lo = int(b) * block_k
        pieces.append(n_spec + np.arange(lo, min(lo + block_k, tp), dtype=np.int64))
    return np.concatenate(pieces)


def sparse_attention_port(q, k, v, frames, patches, specials, mask, block_q, block_k,
                          specials_first=True, panel_blocks=32, threads=None,
                          inputs_permuted=False, work=None):
    """fp32 numpy restatement of sparse_attention (sparse.py:157-205).

    Streams the special-key strip and then the selected key blocks in
    ascending order, ``panel_blocks`` blocks per matmul, merging with the
    online-softmax update of sparse.py:89-98.  ``work`` optionally restricts
    the computation to a list of (head, q_block) items (q_block -1 = the
    special rows); rows outside it are left as NaN (row-sampled timing).
    """
    q, k, v = _f32c(q), _f32c(k), _f32c(v)
    h, n, d = q.shape
    n_spec = frames * specials
    tp = frames * patches
    scale = np.float32(head_scale(d))
    if not inputs_permuted:
        perm, inv = partition_perm(frames, patches, specials, specials_first)
        q, k, v = q[:, perm], k[:, perm], v[:, perm]
    nq = -(-tp // block_q)
    out = np.full((h, n, d), np.nan, dtype=np.float32)
    if work is None:
        work = [(hh, qb) for hh in range(h) for qb in range(-1 if n_spec else 0, nq)]

    def one(item):
        hh, qb = item
        qh, kh, vh = q[hh], k[hh], v[hh]
        if qb < 0:
            # special rows: exact dense softmax over all keys (sparse.py:122-131)
            for r0 in range(0, n_spec, 256):
                r1 = min(r0 + 256, n_spec)
                s = (qh[r0:r1] @ kh.T) * scale
                s -= s.max(axis=1, keepdims=True)
                np.exp(s, out=s)
                s /= s.sum(axis=1, keepdims=True)
                out[hh, r0:r1] = s @ vh
            return
        r0 = n_spec + qb * block_q
        r1 = min(r0 + block_q, n)
        rows = qh[r0:r1]
        m = np.full(rows.shape[0], -np.inf, dtype=np.float32)
        l = np.zeros(rows.shape[0], dtype=np.float32)
        o = np.zeros((rows.shape[0], d), dtype=np.float32)
        panels = []
        if n_spec:
            panels.append(np.arange(n_spec, dtype=np.int64))
        blocks = np.flatnonzero(mask[hh, qb])
        if blocks.size == 0:
            raise ValueError("patch row with empty key-block selection reached the kernel")
        for p0 in range(0, blocks.size, panel_blocks):
            sel = blocks[p0:p0 + panel_blocks]
            idx = (sel[:, None] * block_k + np.arange(block_k)[None, :]).ravel()
            panels.append(n_spec + idx[idx < tp])
        for keys in panels:
            s = (rows @ kh[keys].T) * scale
            m_new = np.maximum(m, s.max(axis=1))
            alpha = np.exp(m - m_new)
            p = np.exp(s - m_new[:, None])
            l *= alpha
            l += p.sum(axis=1)
            o *= alpha[:, None]
            o += p @ vh[keys]
            m = m_new
        out[hh, r0:r1] = o / l[:, None]

    nthreads = threads or host_threads()
    if nthreads <= 1:
        for it in work:
            one(it)
    else:
        with ThreadPoolExecutor(max_workers=nthreads) as ex:
            list(ex.map(one, work))
    if inputs_permuted:
        return out
    return out[:, inv]


def masked_attention_f64(q, k, v, frames, patches, specials, mask, block_q, block_k,
                         specials_first=True, rows=None):
    """Exact float64 softmax attention restricted to the allowed keys.

    Specials see every key; patch queries see every special key plus the
    patch tokens of their q-block's selected key blocks (sparse.py:1-16,
    oracle semantics of the reference's tests/oracles.py:45-82).
    ``rows``: optional iterable of source-order token indices to evaluate;
    returns (H, len(rows), d) then, else (H, T, d), float64.
    """
    q = np.asarray(q, dtype=np.float64)
    k = np.asarray(k, dtype=np.float64)
    v = np.asarray(v, dtype=np.float64)
    h, n, d = q.shape
    n_spec = frames * specials
    tp = frames * patches
    perm, inv = partition_perm(frames, patches, specials, specials_first)
    kp_, vp_ = k[:, perm], v[:, perm]
    src_rows = np.arange(n) if rows is None else np.asarray(list(rows), dtype=np.int64)
    out = np.empty((h, src_rows.size, d), dtype=np.float64)
    scale = head_scale(d)
    part = inv[src_rows]
    # rows sharing a key set (all special rows; the rows of one q-block) are
    # evaluated together, <= 128 rows per matrix product
    group = np.where(part < n_spec, -1, (part - n_spec) // block_q)
    for hh in range(h):
        for gq in np.unique(group):
            idx = np.nonzero(group == gq)[0]
            keys = np.arange(n) if gq < 0 else _row_keys(mask[hh, gq], n_spec, tp, block_k)
            kk, vv = kp_[hh, keys], vp_[hh, keys]
            for c0 in range(0, idx.size, 128):
                sel = idx[c0:c0 + 128]
                s = (q[hh, src_rows[sel]] @ kk.T) * scale
                w = np.exp(s - s.max(axis=1, keepdims=True))
                w /= w.sum(axis=1, keepdims=True)
                out[hh, sel] = w @ vv
    return out


def dense_attention_port(q, k, v, row_chunk=256):
    """fp32 dense attention (dense.py:58-76), the CPU dense baseline."""
    q, k, v = _f32c(q), _f32c(k), _f32c(v)
    h, n, d = q.shape
    scale = np.float32(head_scale(d))
    out = np.empty_like(q)
    for hh in range(h):
        for r0 in range(0, n, row_chunk):
            s = (q[hh, r0:r0 + row_chunk] @ k[hh].T) * scale
            s -= s.max(axis=1, keepdims=True)
            np.exp(s, out=s)
            s /= s.sum(axis=1, keepdims=True)
            out[hh, r0:r0 + row_chunk] = s @ v[hh]
    return out


# ---- dense attention-map statistics -----------------
# Checkers for paper_2509_07120_b200.analysis: the reference's
# dense_attention_map (dense.py:79-102) in float64, its quadrant_stats
# (analysis.py:47-74), and the block-granular attention mass at the
# BlockMask geometry.

def attention_map_f64(q, k) -> np.ndarray:
    """Post-softmax map (H, T, T) in float64 (dense.py:79-102)."""
    q = np.asarray(q, dtype=np.float64)
    k = np.asarray(k, dtype=np.float64)
    scale = float(np.float32(head_scale(q.shape[2])))
    out = np.empty((q.shape[0], q.shape[1], k.shape[1]), dtype=np.float64)
    for h in range(q.shape[0]):
        s = (q[h] @ k[h].T) * scale
        s -= s.max(axis=1, keepdims=True)
        e = np.exp(s)
        out[h] = e / e.sum(axis=1, keepdims=True)
    return out


def quadrant_stats_f64(p, frames: int, patches: int, specials: int, specials_first: bool = True):
    """(means, maxes) dicts of (H,) arrays per quadrant, analysis.py:47-74."""
    n = frames * (patches + specials)
    is_special = np.zeros(n, dtype=bool)
    perm, _ = partition_perm(frames, patches, specials, specials_first)
    is_special[perm[:frames * specials]] = True
    groups = {"S2S": (is_special, is_special), "S2P": (is_special, ~is_special),
              "P2S": (~is_special, is_special), "P2P": (~is_special, ~is_special)}
    means, maxes = {}, {}
    for quad, (qs, ks) in groups.items():
        if not qs.any() or not ks.any():
            continue
        sub = p[:, qs][:, :, ks]
        means[quad] = sub.mean(axis=(1, 2))
        maxes[quad] = sub.max(axis=(1, 2))
    return means, maxes


def block_attention_map_f64(p, frames: int, patches: int, specials: int, block_q: int = 128,
                            block_k: int = 64) -> np.ndarray:
    """(H, nq, nk): mean over the rows of each patch q-block of the summed
    probabilities of each patch k-block (partitioned patch order)."""
    pidx = patch_indices(frames, patches, specials)
    pp = p[:, pidx][:, :, pidx]
    tp = len(pidx)
    nq, nk = -(-tp // block_q), -(-tp // block_k)
    out = np.zeros((p.shape[0], nq, nk), dtype=np.float64)
    for a in range(nq):
        rows = pp[:, a * block_q:(a + 1) * block_q]
        for b in range(nk):
            out[:, a, b] = rows[:, :, b * block_k:(b + 1) * block_k].sum(axis=2).mean(axis=1)
    return out
