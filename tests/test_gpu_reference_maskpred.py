"""The reference's mask-predictor tests (/root/reference/pkg/tests/
test_maskpred.py) re-run against this package's GPU scoring: same scenarios
and thresholds, numpy in / numpy out. (Block pooling, the known-answer
selection rows and the nesting properties also run in test_gpu_score.py.)"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def bsa():
    import paper_2509_07120_b200 as m
    return m


def _geom(bsa, n, block_q=128, block_k=64):
    return bsa.BlockGeometry(n, block_q, block_k)


def _norm_rows(rng, shape):
    raw = rng.random(shape).astype(np.float32)
    return raw / raw.sum(axis=2, keepdims=True)


def test_collinear_block_dominates(bsa):
    d = 16
    qp = np.zeros((1, 1, d), dtype=np.float32)
    kp = np.zeros((1, 4, d), dtype=np.float32)
    qp[0, 0, 0] = 40.0
    kp[0, 2, 0] = 40.0
    kp[0, 0, 1] = kp[0, 1, 2] = kp[0, 3, 3] = 1.0
    assert bsa.pooled_scores(qp, kp, head_dim=d)[0, 0, 2] > 0.99


def test_selection_rules(bsa):
    g4 = _geom(bsa, 4, 4, 1)
    one = bsa.select_blocks(np.array([[[0.97, 0.01, 0.01, 0.01]]], np.float32),
                            bsa.MaskPolicy(0.0, 1.0, g4))
    assert one.blocks.sum() == 1 and one.blocks[0, 0, 0]
    tie = bsa.select_blocks(np.array([[[0.25] * 4]], np.float32), bsa.MaskPolicy(0.5, 1.0, g4))
    assert tie.blocks[0, 0].tolist() == [True, True, False, False]
    rng = np.random.default_rng(5)
    s = bsa.pooled_scores(rng.standard_normal((1, 4, 8)).astype(np.float32),
                          rng.standard_normal((1, 6, 8)).astype(np.float32), head_dim=8)
    full = bsa.select_blocks(s, bsa.MaskPolicy(1.0, 1.0, _geom(bsa, 12, 3, 2)))
    assert full.blocks.all()
    np.testing.assert_allclose(full.achieved_sparsity(), 0.0, atol=1e-12)


def test_coverage_meets_tau(bsa):
    rng = np.random.default_rng(6)
    g = _geom(bsa, 60, 12, 5)
    for _ in range(20):
        scores = _norm_rows(rng, (2, 5, 12))
        tau = float(rng.random())
        mask = bsa.select_blocks(scores, bsa.MaskPolicy(tau, 1.0, g))
        covered = np.where(mask.blocks, scores, 0).sum(axis=2)
        assert (covered >= min(tau, 1.0) - 1e-6).all()


def test_cdf_adapts_to_row_concentration(bsa):
    conc = np.array([0.91] + [0.01] * 9, dtype=np.float32)
    unif = np.full(10, 0.1, dtype=np.float32)
    scores = np.stack([conc, unif])[None]
    g = _geom(bsa, 30, 15, 3)
    counts = bsa.select_blocks(scores, bsa.MaskPolicy(0.9, 1.0, g)).blocks[0].sum(axis=1)
    assert counts[0] == 1 and counts[1] == 9
    assert bsa.select_blocks(scores, bsa.MaskPolicy(0.9, 0.6, g)).blocks[0, 0].sum() == 4


def test_count_floor_and_nesting(bsa):
    rng = np.random.default_rng(7)
    scores = _norm_rows(rng, (1, 4, 10))
    for rho in (0.0, 0.3, 0.8, 1.0):
        mask = bsa.select_blocks(scores, bsa.MaskPolicy(0.0, rho, _geom(bsa, 10, 3, 1)))
        assert (mask.blocks.sum(axis=2) >= min(10, max(1, int(10 * (1 - rho))))).all()
    rng = np.random.default_rng(8)
    scores = _norm_rows(rng, (2, 6, 16))
    prev = None
    for tau in sorted(rng.random(4)):
        m = bsa.select_blocks(scores, bsa.MaskPolicy(float(tau), 0.9, _geom(bsa, 16, 3, 1))).blocks
        if prev is not None:
            assert (m | prev).sum() == m.sum()
        prev = m


def test_sparsity_granularity_bound(bsa):
    rng = np.random.default_rng(10)
    g = _geom(bsa, 530)
    scores = _norm_rows(rng, (2, g.nq_blocks, g.nk_blocks))
    for rho in (0.25, 0.5, 0.9):
        pol = bsa.MaskPolicy(0.0, rho, g)
        mask = bsa.select_blocks(scores, pol)
        bound = (g.nk_blocks - pol.min_blocks) * g.block_k / 530
        assert (mask.achieved_sparsity() <= bound + 1e-12).all()


@pytest.mark.parametrize("rho,tau", [(0.10, 0.97), (0.80, 0.40)])
def test_operating_points(bsa, rho, tau):
    rng = np.random.default_rng(21)
    g = _geom(bsa, 4096)
    q, k = (rng.standard_normal((2, 4096, 64)).astype(np.float32) for _ in range(2))
    sp = bsa.predict_mask(q, k, bsa.MaskPolicy(tau, rho, g)).achieved_sparsity()
    assert (sp <= rho + 1 / g.nk_blocks).all() and (sp >= 0).all()
    if (rho, tau) == (0.80, 0.40):
        rng = np.random.default_rng(22)
        q, k = (rng.standard_normal((1, 4096, 64)).astype(np.float32) for _ in range(2))
        assert bsa.predict_mask(q, k, bsa.MaskPolicy(0.4, 0.8, g)).achieved_sparsity()[0] > 0.3


def test_policy_and_mask_validation(bsa, tmp_path):
    g = _geom(bsa, 64)
    for tau, rho in ((-0.1, 0.5), (0.5, 1.5)):
        with pytest.raises(ValueError):
            bsa.MaskPolicy(tau, rho, g)
    g100 = _geom(bsa, 100, 10, 1)
    assert [bsa.MaskPolicy(0, r, g100).min_blocks for r in (0.75, 1.0, 0.0, 0.9)] == \
        [25, 1, 100, 10]
    g2 = _geom(bsa, 64, 32, 16)
    blocks = np.ones((1, g2.nq_blocks, g2.nk_blocks), dtype=bool)
    blocks[0, 1] = False
    with pytest.raises(ValueError, match="at least one"):
        bsa.BlockMask(blocks, g2)
    path = tmp_path / "m.bsm"
    bsa.write_mask(path, bsa.full_mask(g2, heads=1))
    with pytest.raises(ValueError):
        bsa.read_mask(path, _geom(bsa, 128, 32, 16))


def test_predict_mask_shapes_and_token_check(bsa):
    rng = np.random.default_rng(12)
    g = _geom(bsa, 257)
    q, k = (rng.standard_normal((2, 257, 32)).astype(np.float32) for _ in range(2))
    mask = bsa.predict_mask(q, k, bsa.MaskPolicy(0.5, 0.5, g))
    assert mask.blocks.shape == (2, g.nq_blocks, g.nk_blocks)
    assert mask.blocks.any(axis=2).all()
    q = rng.standard_normal((1, 100, 8)).astype(np.float32)
    with pytest.raises(ValueError, match="patch tokens"):
        bsa.predict_mask(q, q, bsa.MaskPolicy(0.5, 0.5, _geom(bsa, 99)))


def test_row_softmax_reference_cases(bsa):
    """test_tensorio.py TestRowSoftmax of the reference."""
    np.testing.assert_allclose(bsa.row_softmax(np.zeros((1, 4), np.float32)), [[0.25] * 4],
                               atol=1e-7)
    out = bsa.row_softmax(np.array([[1000.0, 0.0]], np.float32))
    np.testing.assert_allclose(out, [[1.0, 0.0]], atol=1e-6)
    assert np.isfinite(out).all()
    rng = np.random.default_rng(3)
    out = bsa.row_softmax(rng.standard_normal((4, 6)).astype(np.float32), scale=0.37)
    np.testing.assert_allclose(out.sum(axis=1), np.ones(4), atol=1e-6)
    assert (out >= 0).all() and (out <= 1).all()
    expected = np.exp([6.0, 0.0]) / np.exp([6.0, 0.0]).sum()
    np.testing.assert_allclose(bsa.row_softmax(np.array([[2.0, 0.0]], np.float32), scale=3.0)[0],
                               expected, atol=1e-6)
