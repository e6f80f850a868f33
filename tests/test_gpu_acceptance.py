"""The reference's acceptance criteria (SPEC.md:422-432,
/root/reference/pkg/tests/test_acceptance.py) on the B200 path.

Numpy in -> numpy out, as in the reference: fp32 inputs run the CUDA-core
kernel (fp32 math). The tolerances are the reference's own: 1e-5 max-abs vs
float64 oracles. C6 runs on the reference's planted-match scene: the
generator is restated in tests/golden_inputs.py and pinned to the
reference's own q/k/v digests (tests/golden/c6_scene.npz, written by
make_golden.py). C7 is the performance gate, run on bf16 inputs as the B200
bench does.
"""

import time

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def bsa():
    import paper_2509_07120_b200 as m
    return m


@pytest.fixture(scope="module")
def oracle():
    import oracle as o
    return o


def gaussian(rng, h, n, d):
    return [rng.standard_normal((h, n, d)).astype(np.float32) for _ in range(3)]


def random_mask(bsa, rng, g, heads, keep):
    blocks = rng.random((heads, g.nq_blocks, g.nk_blocks)) < keep
    empty = ~blocks.any(axis=2)
    if empty.any():
        hi, qi = np.nonzero(empty)
        blocks[hi, qi, rng.integers(g.nk_blocks, size=hi.size)] = True
    return bsa.BlockMask(blocks, g)


def test_c1_zero_sparsity_equals_dense(bsa):
    start = time.perf_counter()
    for heads in (1, 4):
        for n in (257, 1024, 2048):
            rng = np.random.default_rng(1000 + heads * 7 + n)
            q, k, v = gaussian(rng, heads, n, 64)
            inp = bsa.AttentionInputs(q, k, v)
            lay = bsa.TokenLayout(1, n, 0)
            g = bsa.BlockGeometry(n, 128, 64)
            out = bsa.sparse_attention(bsa.SparseAttentionJob(inp, lay, bsa.full_mask(g, heads)))
            err = np.abs(out - bsa.dense_attention(inp)).max()
            assert err <= 1e-5, f"H={heads} N={n}: max abs err {err}"
    assert time.perf_counter() - start < 10.0


def test_c2_masked_oracle_50_random_masks(bsa, oracle):
    rng = np.random.default_rng(2)
    for trial in range(50):
        if trial < 48:
            frames, patches = int(rng.integers(1, 4)), int(rng.integers(40, 180))
            specials = int(rng.choice([0, 3, 5]))
        else:
            frames, patches, specials = 2, 1019, 5
        lay = bsa.TokenLayout(frames, patches, specials)
        heads = int(rng.choice([1, 2]))
        q, k, v = gaussian(rng, heads, lay.total_tokens, 16)
        bq, bk = (int(x) for x in rng.choice([[48, 16], [32, 32], [64, 64]]))
        g = bsa.BlockGeometry(lay.patch_tokens, bq, bk)
        mask = random_mask(bsa, rng, g, heads, float(rng.uniform(0.15, 0.9)))
        out = bsa.sparse_attention(bsa.SparseAttentionJob(bsa.AttentionInputs(q, k, v), lay, mask))
        ref = oracle.masked_attention_f64(q, k, v, frames, patches, specials, mask.blocks, bq, bk)
        err = np.abs(out - ref).max()
        assert err <= 1e-5, f"trial {trial}: max abs err {err}"


def test_c3_selection_rule_exactness(bsa):
    scores = np.array([[[0.5, 0.3, 0.15, 0.05]]], dtype=np.float32)
    g4 = bsa.BlockGeometry(4, block_q=4, block_k=1)
    mask = bsa.select_blocks(scores, bsa.MaskPolicy(0.9, 1.0, g4))
    assert set(np.flatnonzero(mask.blocks[0, 0]).tolist()) == {0, 1, 2}
    rng = np.random.default_rng(3)
    raw = rng.random((2, 5, 100)).astype(np.float32)
    scores = raw / raw.sum(axis=2, keepdims=True)
    g100 = bsa.BlockGeometry(100, block_q=20, block_k=1)
    mask = bsa.select_blocks(scores, bsa.MaskPolicy(0.0, 0.75, g100))
    assert (mask.blocks.sum(axis=2) == 25).all()
    for h in range(2):
        for row in range(5):
            expected = set(np.argsort(-scores[h, row], kind="stable")[:25].tolist())
            assert set(np.flatnonzero(mask.blocks[h, row]).tolist()) == expected


def test_c4_superset_monotonicity(bsa):
    rng = np.random.default_rng(4)
    for trial in range(100):
        nq, nk = int(rng.integers(2, 8)), int(rng.integers(4, 32))
        raw = rng.random((1, nq, nk)).astype(np.float32) ** 3
        scores = raw / raw.sum(axis=2, keepdims=True)
        g = bsa.BlockGeometry(nq * nk, block_q=nk, block_k=nq)
        t1, t2 = sorted(rng.random(2))
        rho = float(rng.random())
        lo = bsa.select_blocks(scores, bsa.MaskPolicy(t2, rho, g))
        hi = bsa.select_blocks(scores, bsa.MaskPolicy(t1, rho, g))
        assert not (hi.blocks & ~lo.blocks).any(), f"trial {trial}: tau nesting"
        r1, r2 = sorted(rng.random(2))
        tau = float(rng.random())
        big = bsa.select_blocks(scores, bsa.MaskPolicy(tau, r1, g))
        small = bsa.select_blocks(scores, bsa.MaskPolicy(tau, r2, g))
        assert not (small.blocks & ~big.blocks).any(), f"trial {trial}: rho nesting"


def test_c5_special_rows_exact_and_carve_out_ablation(bsa):
    rng = np.random.default_rng(5)
    carve_errs, naive_errs = [], []
    for trial in range(40):
        frames, patches = int(rng.integers(1, 4)), int(rng.integers(40, 100))
        lay = bsa.TokenLayout(frames, patches, 5)
        heads, d = int(rng.choice([1, 2])), int(rng.choice([16, 32]))
        q, k, v = gaussian(rng, heads, lay.total_tokens, d)
        inp = bsa.AttentionInputs(q, k, v)
        dense = bsa.dense_attention(inp)
        sidx, pidx = bsa.special_token_indices(lay), bsa.patch_token_indices(lay)
        g = bsa.BlockGeometry(lay.patch_tokens, 32, 16)
        pol = bsa.MaskPolicy(0.0, 0.6, g)
        mask = bsa.predict_mask(q[:, pidx], k[:, pidx], pol)
        out = bsa.sparse_attention(bsa.SparseAttentionJob(inp, lay, mask, pol))
        carve = float(np.abs(out[:, sidx] - dense[:, sidx]).max())
        assert carve <= 1e-5, f"trial {trial}: special-row err {carve}"
        carve_errs.append(carve)
        if trial < 15:
            flat = bsa.TokenLayout(1, lay.total_tokens, 0)
            fg = bsa.BlockGeometry(flat.patch_tokens, 32, 16)
            fmask = bsa.predict_mask(q, k, bsa.MaskPolicy(0.0, 0.6, fg))
            fout = bsa.sparse_attention(bsa.SparseAttentionJob(inp, flat, fmask))
            naive = float(np.abs(fout[:, sidx] - dense[:, sidx]).max())
            assert naive > carve, f"trial {trial}: ablation not worse"
            naive_errs.append(naive)
    assert np.mean(naive_errs) > 10 * max(np.mean(carve_errs), 1e-7)


def _golden_c6():
    import os
    return np.load(os.path.join(os.path.dirname(__file__), "golden", "c6_scene.npz"))


def _sha(a):
    import hashlib
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def test_c6_graceful_degradation(bsa, oracle):
    """C6 (test_acceptance.py:188-206): on the planted-match scene the mean
    per-row relative error against dense attention grows monotonically with
    rho and stays <= 5% at 50% sparsity. Masks are the reference's bit for
    bit; the errors match the reference's own on the fp32 path, and the
    bf16 tensor-core path meets the same criterion."""
    import torch
    from golden_inputs import C6_RHOS, C6_SCENE, c6_inputs

    z = _golden_c6()
    q, k, v = c6_inputs()
    assert (_sha(q), _sha(k), _sha(v)) == (str(z["q_sha"]), str(z["k_sha"]), str(z["v_sha"]))
    n = C6_SCENE["frames"] * C6_SCENE["patches"]
    lay = bsa.TokenLayout(C6_SCENE["frames"], C6_SCENE["patches"], 0)
    g = bsa.BlockGeometry(n, 128, 64)
    dense = oracle.masked_attention_f64(q, k, v, lay.frames, lay.patches_per_frame, 0,
                                        np.ones((1, g.nq_blocks, g.nk_blocks), dtype=bool), 128, 64)
    qb, kb, vb = (torch.from_numpy(x).to("cuda", torch.bfloat16) for x in (q, k, v))
    errs32, errs16 = [], []
    for i, rho in enumerate(C6_RHOS):
        pol = bsa.MaskPolicy(0.0, rho, g)
        mask = bsa.predict_mask(q, k, pol)
        assert np.array_equal(mask.device_bits().cpu().numpy(), z[f"mask{i}_bits"])
        assert mask.achieved_sparsity()[0] == pytest.approx(rho, abs=1e-9)
        out = bsa.sparse_attention(bsa.SparseAttentionJob(bsa.AttentionInputs(q, k, v), lay, mask))
        rel = np.linalg.norm(out - dense, axis=2) / np.linalg.norm(dense, axis=2)
        errs32.append(float(rel.mean()))
        o16 = bsa.sparse_attention(bsa.SparseAttentionJob(bsa.AttentionInputs(qb, kb, vb), lay,
                                                          mask)).float().cpu().numpy()
        rel16 = np.linalg.norm(o16 - dense, axis=2) / np.linalg.norm(dense, axis=2)
        errs16.append(float(rel16.mean()))
    ref = [float(z[f"err{i}"]) for i in range(3)]
    np.testing.assert_allclose(errs32, ref, rtol=1e-4)
    for errs in (errs32, errs16):
        assert errs[0] < errs[1] < errs[2], errs
        assert errs[1] <= 0.05, errs


def test_ragged_cdf_mask_on_planted_scene(bsa, oracle):
    """tau=0.9, rho=0.5 on the C6 scene gives ragged per-row block counts
    (32-49 of 64): the reference's mask bit for bit, and the LPT-scheduled
    tensor-core kernel against the float64 oracle."""
    import torch
    from golden_inputs import C6_SCENE, c6_inputs

    z = _golden_c6()
    q, k, v = c6_inputs()
    lay = bsa.TokenLayout(C6_SCENE["frames"], C6_SCENE["patches"], 0)
    g = bsa.BlockGeometry(lay.patch_tokens, 128, 64)
    mask = bsa.predict_mask(q, k, bsa.MaskPolicy(0.9, 0.5, g))
    assert np.array_equal(mask.device_bits().cpu().numpy(), z["cdf_bits"])
    counts = mask.device_counts().cpu().numpy()
    assert counts.max() - counts.min() >= 8, "expected ragged rows"
    qb, kb, vb = (torch.from_numpy(x).to("cuda", torch.bfloat16) for x in (q, k, v))
    out = bsa.sparse_attention(bsa.SparseAttentionJob(bsa.AttentionInputs(qb, kb, vb), lay, mask))
    ref = oracle.masked_attention_f64(*(t.float().cpu().numpy() for t in (qb, kb, vb)),
                                      lay.frames, lay.patches_per_frame, 0, mask.blocks, 128, 64)
    o = out.float().cpu().numpy()
    assert float(np.abs(o - ref).max() / np.abs(ref).max()) <= 2e-2


def test_c7_performance_gate_and_flop_accounting(bsa):
    from paper_2509_07120_b200.benchsweep import bench_inputs, bench_sweep
    # 16 heads instead of the reference's 1: one head of 32K tokens is a few
    # hundred microseconds on a B200, launch-bound, and would not show the
    # quadratic regime the gate checks
    rows = bench_sweep([16384, 32768], 0.0, 0.75, repeats=3, head_dim=64, heads=16, seed=0)
    big = rows[1]
    assert big.achieved_sparsity >= 0.70
    assert big.sparse_ms <= 0.5 * big.dense_ms, f"sparse {big.sparse_ms} vs dense {big.dense_ms}"
    assert rows[1].dense_ms / rows[0].dense_ms >= 3.0
    inputs, lay = bench_inputs(32768, 64, 1, 0)
    pol = bsa.MaskPolicy(0.0, 0.75, bsa.BlockGeometry(32768, 128, 64))
    mask = bsa.predict_mask(inputs.q, inputs.k, pol)
    est = bsa.flop_estimate(bsa.SparseAttentionJob(inputs, lay, mask, pol))
    bound = 1.0 / (1.0 - float(mask.achieved_sparsity()[0]))
    assert abs(est.theoretical_speedup - bound) / bound <= 0.05


def test_c9_bit_identical_files_across_runs(bsa, tmp_path):
    rng = np.random.default_rng(11)
    q, k, v = gaussian(rng, 1, 512, 32)
    lay = bsa.TokenLayout(2, 256, 0)
    g = bsa.BlockGeometry(512, 64, 32)
    pol = bsa.MaskPolicy(0.5, 0.5, g)
    arts = []
    for run in "ab":
        mask = bsa.predict_mask(q, k, pol)
        bsa.write_mask(tmp_path / f"{run}.bsm", mask)
        out = bsa.sparse_attention(bsa.SparseAttentionJob(bsa.AttentionInputs(q, k, v), lay, mask, pol))
        bsa.write_tensor(tmp_path / f"{run}.bsat", out)
        arts.append(((tmp_path / f"{run}.bsm").read_bytes(), (tmp_path / f"{run}.bsat").read_bytes()))
    assert arts[0] == arts[1]
    np.testing.assert_array_equal(bsa.read_mask(tmp_path / "a.bsm", g).blocks,
                                  bsa.read_mask(tmp_path / "b.bsm", g).blocks)
