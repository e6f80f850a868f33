"""The reference's block-sparse kernel tests (/root/reference/pkg/tests/
test_sparse.py) re-run against this package: same scenarios, same
tolerances, numpy in / numpy out (fp32 inputs: the CUDA-core fp32 path).
The masked-dense checker is the float64 oracle (oracle/)."""

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def bsa():
    import paper_2509_07120_b200 as m
    return m


def _inputs(bsa, h, n, d, seed):
    rng = np.random.default_rng(seed)
    return bsa.AttentionInputs(*(rng.standard_normal((h, n, d)).astype(np.float32)
                                 for _ in range(3)))


def _random_mask(bsa, rng, g, heads, keep=0.5):
    blocks = rng.random((heads, g.nq_blocks, g.nk_blocks)) < keep
    empty = ~blocks.any(axis=2)
    if empty.any():
        hi, qi = np.nonzero(empty)
        blocks[hi, qi, rng.integers(g.nk_blocks, size=hi.size)] = True
    return bsa.BlockMask(blocks, g)


@pytest.mark.parametrize("n", [64, 257, 400])
@pytest.mark.parametrize("heads", [1, 2])
def test_full_mask_no_specials_equals_dense(bsa, n, heads):
    inp = _inputs(bsa, heads, n, 32, n + heads)
    lay = bsa.TokenLayout(frames=1, patches_per_frame=n, specials_per_frame=0)
    job = bsa.SparseAttentionJob(inp, lay, bsa.full_mask(bsa.BlockGeometry(n, 128, 64), heads))
    np.testing.assert_allclose(bsa.sparse_attention(job), bsa.dense_attention(inp), atol=1e-5)


def test_full_mask_with_specials_equals_dense(bsa):
    lay = bsa.TokenLayout(frames=3, patches_per_frame=90, specials_per_frame=5)
    inp = _inputs(bsa, 2, lay.total_tokens, 16, 42)
    job = bsa.SparseAttentionJob(inp, lay,
                                 bsa.full_mask(bsa.BlockGeometry(lay.patch_tokens, 32, 16), 2))
    np.testing.assert_allclose(bsa.sparse_attention(job), bsa.dense_attention(inp), atol=1e-5)


def _job(bsa, seed):
    rng = np.random.default_rng(seed)
    lay = bsa.TokenLayout(frames=2, patches_per_frame=130, specials_per_frame=4)
    inp = _inputs(bsa, 2, lay.total_tokens, 16, seed)
    g = bsa.BlockGeometry(lay.patch_tokens, 64, 16)
    return bsa.SparseAttentionJob(inp, lay, _random_mask(bsa, rng, g, 2))


def test_random_masks_vs_masked_dense_oracle(bsa):
    for seed in range(4):
        job = _job(bsa, seed)
        lay = job.layout
        ref = oracle.masked_attention_f64(job.inputs.q.cpu().numpy(), job.inputs.k.cpu().numpy(),
                                          job.inputs.v.cpu().numpy(), lay.frames,
                                          lay.patches_per_frame, lay.specials_per_frame,
                                          job.mask.blocks, 64, 16)
        np.testing.assert_allclose(bsa.sparse_attention(job), ref, atol=1e-5)


def test_panel_grouping_and_threads_are_irrelevant(bsa):
    job = _job(bsa, 5)
    base = bsa.sparse_attention(job, panel_blocks=1)
    for pb in (2, 5, 32):
        assert bsa.sparse_attention(job, panel_blocks=pb).tobytes() == base.tobytes()
    assert bsa.sparse_attention(job, threads=3).tobytes() == base.tobytes()
    assert bsa.sparse_attention(job).tobytes() == base.tobytes()


def test_mismatches_rejected(bsa):
    lay = bsa.TokenLayout(frames=1, patches_per_frame=64, specials_per_frame=0)
    with pytest.raises(ValueError, match="patch tokens"):
        bsa.SparseAttentionJob(_inputs(bsa, 1, 64, 8, 9), lay,
                               bsa.full_mask(bsa.BlockGeometry(96, 32, 16), 1))
    with pytest.raises(ValueError, match="heads"):
        bsa.SparseAttentionJob(_inputs(bsa, 2, 64, 8, 10), lay,
                               bsa.full_mask(bsa.BlockGeometry(64, 32, 16), 1))


def test_stats_reports_match_plain_kernel(bsa):
    job = _job(bsa, 11)
    plain = bsa.sparse_attention(job)
    out, reports = bsa.sparse_attention_stats(job)
    assert np.asarray(out).tobytes() == plain.tobytes()
    sp = job.mask.achieved_sparsity()
    assert len(reports) == 2
    for r in reports:
        assert r.achieved_sparsity == pytest.approx(float(sp[r.head]))
        assert r.wall_ms >= 0 and r.theoretical_speedup > 1.0


def test_flop_accounting(bsa):
    lay = bsa.TokenLayout(frames=2, patches_per_frame=64, specials_per_frame=3)
    job = bsa.SparseAttentionJob(_inputs(bsa, 2, lay.total_tokens, 8, 12), lay,
                                 bsa.full_mask(bsa.BlockGeometry(lay.patch_tokens, 32, 16), 2))
    est = bsa.flop_estimate(job)
    assert est.dense_flops == est.sparse_flops and est.theoretical_speedup == pytest.approx(1.0)
    n = 4096
    lay = bsa.TokenLayout(frames=1, patches_per_frame=n, specials_per_frame=0)
    g = bsa.BlockGeometry(n, 128, 64)
    blocks = np.zeros((1, g.nq_blocks, g.nk_blocks), dtype=bool)
    blocks[:, :, :16] = True
    job = bsa.SparseAttentionJob(_inputs(bsa, 1, n, 8, 13), lay, bsa.BlockMask(blocks, g))
    assert bsa.flop_estimate(job).theoretical_speedup == pytest.approx(4.0)
    assert job.mask.achieved_sparsity()[0] == pytest.approx(0.75)
    # closed form vs direct enumeration of allowed (query, key) pairs
    rng = np.random.default_rng(14)
    lay = bsa.TokenLayout(frames=2, patches_per_frame=64, specials_per_frame=1)
    g = bsa.BlockGeometry(lay.patch_tokens, 32, 16)
    mask = _random_mask(bsa, rng, g, 1)
    job = bsa.SparseAttentionJob(_inputs(bsa, 1, lay.total_tokens, 8, 15), lay, mask)
    ns, tp = lay.special_tokens, lay.patch_tokens
    allowed = ns * lay.total_tokens  # special rows see everything
    for r in range(tp):
        qb = r // 32
        keys = ns + sum(min(16, tp - kb * 16) for kb in np.flatnonzero(mask.blocks[0, qb]))
        allowed += keys
    est = bsa.flop_estimate(job)
    assert est.sparse_flops == 2 * 8 * allowed
    assert est.dense_flops == 2 * 8 * lay.total_tokens ** 2
