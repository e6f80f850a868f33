"""Generate golden fixtures by running the REFERENCE package in this container.

    PYTHONDONTWRITEBYTECODE=1 PYTHONPATH=/root/reference/pkg/src \
        python tests/golden/make_golden.py

The reference (/root/reference/pkg/src/bsattn, numpy + OpenBLAS) does not
exist on the GPU box, so its outputs are committed here as small .npz files.
Inputs are never stored: every case is regenerated from a numpy PCG64 seed
exactly as the reference's own tests and bench do (bench.py:46-70,
test_sparse.py:15-21): ``default_rng(seed).standard_normal((H, T, d))`` for
q, k, v in that order, cast to float32.  ``tests/golden_inputs.py`` holds the
shared regeneration code.
"""

from __future__ import annotations

import hashlib
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))  # tests/

from golden_inputs import (  # noqa: E402
    C6_RHOS,
    C6_SCENE,
    CASES_ATTN,
    CASES_FULL,
    FULL_POLICIES,
    CASES_MAP,
    CASES_SCORE,
    SCORE_POLICIES,
    bf16_round,
    make_qkv,
    c6_inputs,
    sample_rows,
)

import bsattn  # noqa: E402  (the reference, via PYTHONPATH)
from bsattn import (  # noqa: E402
    AttentionInputs,
    BlockGeometry,
    MaskPolicy,
    SparseAttentionJob,
    TokenLayout,
    patch_token_indices,
    predict_mask,
    sparse_attention,
)
from bsattn.analysis import quadrant_stats  # noqa: E402
from bsattn.dense import dense_attention_map  # noqa: E402
from bsattn.maskpred import block_pool, pooled_scores, select_blocks  # noqa: E402


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def score_case(name, frames, patches, specials, heads, d, seed, block_q, block_k):
    t0 = time.time()
    lay = TokenLayout(frames, patches, specials)
    q, k, _ = make_qkv(heads, lay.total_tokens, d, seed)
    pidx = patch_token_indices(lay)
    qp_in, kp_in = np.ascontiguousarray(q[:, pidx]), np.ascontiguousarray(k[:, pidx])
    g = BlockGeometry(lay.patch_tokens, block_q, block_k)
    qp = block_pool(qp_in, block_q)
    kp = block_pool(kp_in, block_k)
    probs = pooled_scores(qp, kp, d)
    out = dict(
        frames=frames, patches=patches, specials=specials, heads=heads, d=d, seed=seed,
        block_q=block_q, block_k=block_k,
        qp_sha=sha(qp), kp_sha=sha(kp), probs_sha=sha(probs),
        probs_head0=probs[0, :16],
        qp_head0=qp[0, :16], kp_head0=kp[0, :32],
    )
    for i, (tau, rho) in enumerate(SCORE_POLICIES):
        m = select_blocks(probs, MaskPolicy(tau, rho, g)).blocks
        out[f"mask{i}_bits"] = np.packbits(m.reshape(-1, m.shape[2]), axis=1, bitorder="little")
        out[f"mask{i}_tau_rho"] = np.array([tau, rho])
    np.savez_compressed(os.path.join(HERE, f"score_{name}.npz"), **out)
    print(f"score_{name}: nq={g.nq_blocks} nk={g.nk_blocks} ({time.time() - t0:.1f}s)")


def full_case(name, frames, patches, specials, heads, d, seed, bf16):
    """Headline size: digests of the reference's pooled Q/K, probabilities and
    masks (two policies) plus the per-row selected-block counts."""
    t0 = time.time()
    lay = TokenLayout(frames, patches, specials)
    q, k, _ = make_qkv(heads, lay.total_tokens, d, seed)
    if bf16:
        q, k = bf16_round(q), bf16_round(k)
    pidx = patch_token_indices(lay)
    qp_in, kp_in = np.ascontiguousarray(q[:, pidx]), np.ascontiguousarray(k[:, pidx])
    g = BlockGeometry(lay.patch_tokens, 128, 64)
    qp, kp = block_pool(qp_in, 128), block_pool(kp_in, 64)
    probs = pooled_scores(qp, kp, d)
    out = dict(frames=frames, patches=patches, specials=specials, heads=heads, d=d, seed=seed,
               bf16=bf16, qp_sha=sha(qp), kp_sha=sha(kp), probs_sha=sha(probs))
    for i, (tau, rho) in enumerate(FULL_POLICIES):
        m = predict_mask(qp_in, kp_in, MaskPolicy(tau, rho, g)).blocks
        bits = np.packbits(m.reshape(-1, m.shape[2]), axis=1, bitorder="little")
        out[f"mask{i}_sha"] = sha(bits)
        out[f"mask{i}_counts"] = m.sum(axis=2).astype(np.uint16)
        out[f"mask{i}_tau_rho"] = np.array([tau, rho])
    np.savez_compressed(os.path.join(HERE, f"full_{name}.npz"), **out)
    print(f"full_{name}: nq={g.nq_blocks} nk={g.nk_blocks} ({time.time() - t0:.1f}s)")


def attn_case(name, frames, patches, specials, heads, d, seed, block_q, block_k, tau, rho,
              full=True):
    t0 = time.time()
    lay = TokenLayout(frames, patches, specials)
    q, k, v = make_qkv(heads, lay.total_tokens, d, seed)
    pidx = patch_token_indices(lay)
    g = BlockGeometry(lay.patch_tokens, block_q, block_k)
    mask = predict_mask(q[:, pidx], k[:, pidx], MaskPolicy(tau, rho, g))
    job = SparseAttentionJob(AttentionInputs(q, k, v), lay, mask)
    o = sparse_attention(job, threads=os.cpu_count() or 1)
    out = dict(
        frames=frames, patches=patches, specials=specials, heads=heads, d=d, seed=seed,
        block_q=block_q, block_k=block_k, tau=tau, rho=rho,
        mask_bits=np.packbits(mask.blocks.reshape(-1, g.nk_blocks), axis=1, bitorder="little"),
        out_sum=np.float64(o.astype(np.float64).sum()),
        out_abs_sum=np.float64(np.abs(o.astype(np.float64)).sum()),
    )
    if full:
        out["out"] = o
    else:
        rows = sample_rows(lay, block_q)
        out["rows"] = rows
        out["out_rows"] = o[:, rows]
    np.savez_compressed(os.path.join(HERE, f"attn_{name}.npz"), **out)
    print(f"attn_{name}: T={lay.total_tokens} ({time.time() - t0:.1f}s)")


def map_case(name, frames, patches, specials, heads, d, seed):
    """Reference dense_attention_map (dense.py:79-102) + quadrant_stats
    (analysis.py:47-74) on bf16-rounded q/k, and the block-granular mass
    (mean over a 128-row patch q-block of the summed probabilities of a
    64-key patch k-block) of that same reference map."""
    t0 = time.time()
    lay = TokenLayout(frames, patches, specials)
    q, k, v = make_qkv(heads, lay.total_tokens, d, seed)
    q, k = bf16_round(q), bf16_round(k)
    maps = dense_attention_map(AttentionInputs(q, k, v))
    st = quadrant_stats(maps, lay)
    pidx = patch_token_indices(lay)
    pp = maps[:, pidx][:, :, pidx].astype(np.float64)
    tp = lay.patch_tokens
    nq, nk = -(-tp // 128), -(-tp // 64)
    bm = np.zeros((heads, nq, nk), dtype=np.float64)
    for a in range(nq):
        rows = pp[:, a * 128:(a + 1) * 128]
        for b in range(nk):
            bm[:, a, b] = rows[:, :, b * 64:(b + 1) * 64].sum(axis=2).mean(axis=1)
    out = dict(frames=frames, patches=patches, specials=specials, heads=heads, d=d, seed=seed,
               block_map=bm.astype(np.float32), quads=np.array(sorted(st.means)))
    for quad in st.means:
        out[f"mean_{quad}"] = st.means[quad]
        out[f"max_{quad}"] = st.maxes[quad]
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
    print(f"{name}: T={lay.total_tokens} ({time.time() - t0:.1f}s)")


def c6_case():
    """Acceptance C6 scene through the reference itself: its q/k/v digests
    (pinning tests/golden_inputs.py's restatement of synth.py), its masks and
    the mean relative error against dense at each rho."""
    from bsattn.dense import dense_attention
    from bsattn.synth import SynthScene, full_shift_matches, synth_scene

    t0 = time.time()
    s = C6_SCENE
    matches, groups = full_shift_matches(s["frames"], s["patches"], seed=s["match_seed"],
                                         group_length=s["group_length"],
                                         shift_quantum=s["shift_quantum"])
    scene = SynthScene(frames=s["frames"], patches_per_frame=s["patches"], head_dim=s["d"],
                       matches=matches, c=s["c"], direction_groups=groups)
    res = synth_scene(scene, seed=s["seed"])
    q, k, v = res.inputs.q, res.inputs.k, res.inputs.v
    mq, mk, mv = c6_inputs()
    assert sha(q) == sha(mq) and sha(k) == sha(mk) and sha(v) == sha(mv), "restatement drifted"
    dense = dense_attention(res.inputs)
    g = BlockGeometry(s["frames"] * s["patches"], 128, 64)
    out = dict(q_sha=sha(q), k_sha=sha(k), v_sha=sha(v), dense_sha=sha(dense))
    for i, rho in enumerate(C6_RHOS):
        policy = MaskPolicy(tau=0.0, rho=rho, geometry=g)
        mask = predict_mask(q, k, policy)
        o = sparse_attention(SparseAttentionJob(res.inputs, scene.layout, mask, policy))
        rel = np.linalg.norm(o - dense, axis=2) / np.linalg.norm(dense, axis=2)
        out[f"mask{i}_bits"] = np.packbits(mask.blocks.reshape(-1, g.nk_blocks), axis=1,
                                           bitorder="little")
        out[f"err{i}"] = np.float64(rel.mean())
    # a CDF policy on the same scene: ragged per-row counts (the LPT case)
    mask = predict_mask(q, k, MaskPolicy(tau=0.9, rho=0.5, geometry=g))
    out["cdf_bits"] = np.packbits(mask.blocks.reshape(-1, g.nk_blocks), axis=1, bitorder="little")
    np.savez_compressed(os.path.join(HERE, "c6_scene.npz"), **out)
    print(f"c6_scene: errors {[float(out[f'err{i}']) for i in range(3)]} ({time.time() - t0:.1f}s)")


def main():
    print("reference bsattn", bsattn.__version__, "numpy", np.__version__)
    only = sys.argv[1:]  # optional case names
    for c in CASES_SCORE:
        if not only or c["name"] in only:
            score_case(**c)
    for c in CASES_ATTN:
        if not only or c["name"] in only:
            attn_case(**c)
    for c in CASES_MAP:
        if not only or c["name"] in only:
            map_case(**c)
    for c in CASES_FULL:
        if not only or c["name"] in only:
            full_case(**c)
    if not only or "c6" in only:
        c6_case()


if __name__ == "__main__":
    main()
