"""Scoring stage on the B200 vs the oracle and the reference's golden fixtures.

Bar: bit-exact (pooled means, probabilities and block masks) for fp32
inputs; for bf16 inputs the oracle is fed the bf16-rounded values upcast to
fp32, and the masks must again be bit-exact.
"""

import hashlib
import os

import numpy as np
import pytest

from golden_inputs import CASES_SCORE, SCORE_POLICIES, make_qkv

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.fixture(scope="module")
def bsa():
    import paper_2509_07120_b200 as m
    return m


@pytest.fixture(scope="module")
def oracle():
    import oracle as o
    return o


def _patch_inputs(c):
    import oracle
    q, k, _ = make_qkv(c["heads"], c["frames"] * (c["patches"] + c["specials"]), c["d"], c["seed"])
    pidx = oracle.patch_indices(c["frames"], c["patches"], c["specials"])
    return q, k, pidx


@pytest.mark.parametrize("case", CASES_SCORE, ids=[c["name"] for c in CASES_SCORE])
def test_block_pool_bit_exact(bsa, oracle, case):
    q, k, pidx = _patch_inputs(case)
    for x, blk in ((q, case["block_q"]), (k, case["block_k"])):
        xp = np.ascontiguousarray(x[:, pidx])
        dev = bsa.block_pool(xp, blk)
        ref = oracle.block_pool(xp, blk)
        assert dev.dtype == np.float32 and dev.shape == ref.shape
        assert np.array_equal(dev.view(np.uint32), ref.view(np.uint32))


@pytest.mark.parametrize("case", CASES_SCORE, ids=[c["name"] for c in CASES_SCORE])
def test_predict_mask_matches_golden(bsa, case):
    """Device masks equal the reference's own masks for every policy."""
    z = np.load(os.path.join(GOLDEN, f"score_{case['name']}.npz"))
    q, k, pidx = _patch_inputs(case)
    lay = bsa.TokenLayout(case["frames"], case["patches"], case["specials"])
    g = bsa.BlockGeometry(lay.patch_tokens, case["block_q"], case["block_k"])
    qp, kp = np.ascontiguousarray(q[:, pidx]), np.ascontiguousarray(k[:, pidx])
    for i, (tau, rho) in enumerate(SCORE_POLICIES):
        pol = bsa.MaskPolicy(tau, rho, g)
        m = bsa.predict_mask(qp, kp, pol)
        got = m.device_bits().cpu().numpy()
        assert np.array_equal(got, z[f"mask{i}_bits"]), f"policy {tau},{rho}"
        # gather folded into the kernels: same mask from the interleaved tensors
        m2 = bsa.predict_mask(q, k, pol, layout=lay)
        assert np.array_equal(m2.device_bits().cpu().numpy(), got)
        counts = m.device_counts().cpu().numpy()
        assert np.array_equal(counts, m.blocks.sum(axis=2).reshape(-1))


@pytest.mark.parametrize("case", CASES_SCORE[:2], ids=[c["name"] for c in CASES_SCORE[:2]])
def test_pooled_probabilities_match_golden(bsa, case):
    """At the configs the probability tensors equal the reference's bit for bit."""
    z = np.load(os.path.join(GOLDEN, f"score_{case['name']}.npz"))
    q, k, pidx = _patch_inputs(case)
    qp = bsa.block_pool(np.ascontiguousarray(q[:, pidx]), case["block_q"])
    kp = bsa.block_pool(np.ascontiguousarray(k[:, pidx]), case["block_k"])
    assert sha(qp) == str(z["qp_sha"]) and sha(kp) == str(z["kp_sha"])
    pr = bsa.pooled_scores(qp, kp, case["d"])
    assert sha(pr) == str(z["probs_sha"])


@pytest.mark.parametrize("case", CASES_SCORE, ids=[c["name"] for c in CASES_SCORE])
def test_pooled_scores_vs_oracle(bsa, oracle, case):
    q, k, pidx = _patch_inputs(case)
    qp = oracle.block_pool(q[:, pidx], case["block_q"])
    kp = oracle.block_pool(k[:, pidx], case["block_k"])
    dev = bsa.pooled_scores(qp, kp, case["d"])
    ref = oracle.pooled_scores(qp, kp, case["d"])
    assert np.array_equal(dev.view(np.uint32), ref.view(np.uint32))


def test_bf16_inputs_mask_bit_exact(bsa, oracle):
    import torch
    c = CASES_SCORE[0]
    q, k, pidx = _patch_inputs(c)
    qb = torch.from_numpy(np.ascontiguousarray(q[:, pidx])).to("cuda", torch.bfloat16)
    kb = torch.from_numpy(np.ascontiguousarray(k[:, pidx])).to("cuda", torch.bfloat16)
    g = bsa.BlockGeometry(qb.shape[1], 128, 64)
    for tau, rho in SCORE_POLICIES:
        m = bsa.predict_mask(qb, kb, bsa.MaskPolicy(tau, rho, g))
        ref, _ = oracle.predict_mask(qb.float().cpu().numpy(), kb.float().cpu().numpy(), 128, 64,
                                     tau, rho)
        assert np.array_equal(m.blocks, ref), (tau, rho)


# -------- reference test_maskpred.py behaviours (maskpred.py semantics) --------

def test_select_hand_examples(bsa):
    geom = lambda n, bq, bk: bsa.BlockGeometry(n, bq, bk)  # noqa: E731
    s = np.array([[[0.5, 0.3, 0.15, 0.05]]], dtype=np.float32)
    m = bsa.select_blocks(s, bsa.MaskPolicy(0.9, 1.0, geom(4, 4, 1)))
    assert m.blocks[0, 0].tolist() == [True, True, True, False]
    s = np.array([[[0.97, 0.01, 0.01, 0.01]]], dtype=np.float32)
    m = bsa.select_blocks(s, bsa.MaskPolicy(0.0, 1.0, geom(4, 4, 1)))
    assert m.blocks.sum() == 1 and m.blocks[0, 0, 0]
    s = np.array([[[0.25, 0.25, 0.25, 0.25]]], dtype=np.float32)
    m = bsa.select_blocks(s, bsa.MaskPolicy(0.5, 1.0, geom(4, 4, 1)))
    assert m.blocks[0, 0].tolist() == [True, True, False, False]


def test_select_ratio_floor_is_top_k(bsa, oracle):
    rng = np.random.default_rng(4)
    raw = rng.random((1, 3, 100)).astype(np.float32)
    scores = raw / raw.sum(axis=2, keepdims=True)
    pol = bsa.MaskPolicy(0.0, 0.75, bsa.BlockGeometry(100, 34, 1))
    m = bsa.select_blocks(scores, pol)
    assert (m.blocks.sum(axis=2) == 25).all()
    for row in range(3):
        top = set(np.argsort(-scores[0, row], kind="stable")[:25].tolist())
        assert set(np.flatnonzero(m.blocks[0, row]).tolist()) == top


@pytest.mark.parametrize("seed", range(8))
def test_select_random_policies_vs_oracle(bsa, oracle, seed):
    """Random (tau, rho), peaked and flat rows, ties, tau = 0 and 1."""
    rng = np.random.default_rng(1000 + seed)
    nk = int(rng.integers(1, 300))
    g = bsa.BlockGeometry(nk, int(rng.integers(1, 50)), 1)
    h, nq = 2, g.nq_blocks
    temp = float(rng.choice([0.05, 1.0, 20.0]))
    z = rng.standard_normal((h, nq, nk)) * temp
    if seed % 3 == 0:
        z = np.round(z)  # many exact ties
    p = np.exp(z - z.max(axis=2, keepdims=True))
    p = (p / p.sum(axis=2, keepdims=True)).astype(np.float32)
    for tau in (0.0, float(rng.random()), 0.999, 1.0):
        rho = float(rng.random())
        k_floor = oracle.min_blocks(nk, rho)
        ref, cnt = oracle.select_blocks(p, tau, k_floor)
        m = bsa.select_blocks(p, bsa.MaskPolicy(tau, rho, g))
        assert np.array_equal(m.blocks, ref), (tau, rho, nk)
        assert np.array_equal(m.device_counts().cpu().numpy(), cnt.reshape(-1))


def test_select_unnormalised_and_negative_scores(bsa, oracle):
    """Rows the exact fast path refuses (negative, > 2, tiny) go through the
    sort-based fallback and still match the reference algorithm."""
    rng = np.random.default_rng(7)
    s = rng.standard_normal((1, 5, 40)).astype(np.float32) * 3.0
    s[0, 1] = np.abs(s[0, 1]) * 1e-12
    s[0, 2] = 5.0
    g = bsa.BlockGeometry(40 * 8, 64, 8)
    assert (g.nq_blocks, g.nk_blocks) == (5, 40)
    for tau, rho in ((0.3, 0.9), (1.0, 1.0), (0.0, 0.5)):
        ref, _ = oracle.select_blocks(s, tau, oracle.min_blocks(40, rho))
        m = bsa.select_blocks(s, bsa.MaskPolicy(tau, rho, g))
        assert np.array_equal(m.blocks, ref), (tau, rho)


def test_pool_ragged_and_identity(bsa):
    rng = np.random.default_rng(2)
    x = rng.standard_normal((1, 5, 4)).astype(np.float32)
    out = bsa.block_pool(x, 2)
    assert out.shape == (1, 3, 4)
    np.testing.assert_allclose(out[0, 2], x[0, 4], atol=0)
    x = rng.standard_normal((1, 6, 3)).astype(np.float32)
    np.testing.assert_array_equal(bsa.block_pool(x, 1), x)
    x = rng.standard_normal((2, 9, 5)).astype(np.float32)
    np.testing.assert_allclose(bsa.block_pool(x, 9), x.mean(axis=1, keepdims=True), atol=1e-6)
    with pytest.raises(ValueError):
        bsa.block_pool(np.ones((1, 4, 2), dtype=np.float32), 0)


def test_pool_long_blocks_vs_oracle(bsa, oracle):
    """block > 129 exercises numpy's recursive pairwise split."""
    rng = np.random.default_rng(9)
    x = rng.standard_normal((2, 1000, 12)).astype(np.float32)
    for blk in (130, 257, 600, 1000):
        assert np.array_equal(bsa.block_pool(x, blk), oracle.block_pool(x, blk))


def test_scores_rows_sum_and_uniform(bsa):
    qp = np.ones((1, 3, 8), dtype=np.float32)
    kp = np.ones((1, 5, 8), dtype=np.float32)
    np.testing.assert_allclose(bsa.pooled_scores(qp, kp, 8), np.full((1, 3, 5), 0.2), atol=1e-6)
    d = 16
    qp = np.zeros((1, 1, d), dtype=np.float32)
    kp = np.zeros((1, 4, d), dtype=np.float32)
    qp[0, 0, 0] = 40.0
    kp[0, 2, 0] = 40.0
    assert bsa.pooled_scores(qp, kp, d)[0, 0, 2] > 0.99


def test_row_softmax_bit_exact(bsa, oracle):
    rng = np.random.default_rng(11)
    a = (rng.standard_normal((37, 301)) * 4).astype(np.float32)
    dev = bsa.row_softmax(a, 0.125)
    z = a * np.float32(0.125)
    z = z - z.max(axis=1, keepdims=True)
    e = oracle.np_expf(z)
    ref = e / np.array([[oracle.lib().oracle_pairwise_sum(
        np.ascontiguousarray(r).ctypes.data_as(__import__("ctypes").c_void_p), r.size)]
        for r in e], dtype=np.float32)
    assert np.array_equal(dev, ref.astype(np.float32))
    big = bsa.row_softmax(np.array([[1000.0, 0.0]], dtype=np.float32))
    assert big[0, 0] == 1.0 and big[0, 1] == 0.0


def test_nesting_property(bsa):
    """Masks are nested in tau and in rho (acceptance C4)."""
    rng = np.random.default_rng(21)
    q = rng.standard_normal((2, 2000, 64)).astype(np.float32)
    k = rng.standard_normal((2, 2000, 64)).astype(np.float32)
    g = bsa.BlockGeometry(2000, 128, 64)
    prev = None
    for tau in (0.1, 0.3, 0.5, 0.8, 0.95):
        m = bsa.predict_mask(q, k, bsa.MaskPolicy(tau, 0.9, g)).blocks
        if prev is not None:
            assert (prev <= m).all()
        prev = m
