"""Dense attention-map statistics on the GPU (analysis.py, csrc/bsa_stats_tc.cu)
against fixtures the REFERENCE produced (dense_attention_map +
quadrant_stats, tests/golden/make_golden.py) and the float64 oracle."""

import os

import numpy as np
import pytest

import oracle
from golden_inputs import CASES_MAP, bf16_round, make_qkv

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def bsa():
    import paper_2509_07120_b200 as m
    return m


def _inputs(bsa, c, dtype="bf16"):
    import torch
    T = c["frames"] * (c["patches"] + c["specials"])
    q, k, v = make_qkv(c["heads"], T, c["d"], c["seed"])
    q, k = bf16_round(q), bf16_round(k)
    tt = torch.bfloat16 if dtype == "bf16" else torch.float32
    xs = [torch.from_numpy(x).to("cuda", tt) for x in (q, k, v)]
    return bsa.AttentionInputs(*xs), bsa.TokenLayout(c["frames"], c["patches"], c["specials"])


@pytest.mark.parametrize("c", CASES_MAP, ids=[c["name"] for c in CASES_MAP])
def test_quadrant_stats_and_block_map_vs_reference(bsa, c):
    from paper_2509_07120_b200.analysis import attention_quadrant_stats, block_attention_map

    g = np.load(os.path.join(GOLDEN, f"{c['name']}.npz"))
    for dtype in ("bf16", "f32"):  # f32 inputs are rounded to bf16 (they already are)
        inp, lay = _inputs(bsa, c, dtype)
        st = attention_quadrant_stats(inp, lay)
        assert sorted(st.means) == sorted(str(x) for x in g["quads"])
        for quad in st.means:
            np.testing.assert_allclose(st.means[quad], g[f"mean_{quad}"], rtol=2e-4)
            np.testing.assert_allclose(st.maxes[quad], g[f"max_{quad}"], rtol=2e-4)
        bm = block_attention_map(inp, lay).cpu().numpy()
        np.testing.assert_allclose(bm, g["block_map"], rtol=1e-3, atol=1e-6)


def test_block_map_deterministic_and_recall(bsa):
    import torch
    from paper_2509_07120_b200.analysis import block_attention_map, mask_recall

    c = CASES_MAP[0]
    inp, lay = _inputs(bsa, c)
    a = block_attention_map(inp, lay)
    b = block_attention_map(inp, lay)
    assert torch.equal(a, b)
    g = bsa.BlockGeometry(lay.patch_tokens, 128, 64)
    full = mask_recall(a, bsa.full_mask(g, c["heads"]))
    np.testing.assert_allclose(full.cpu().numpy(), 1.0, rtol=1e-12)
    # nested masks (superset monotonicity, C4) keep nested attention mass
    r = [mask_recall(a, bsa.predict_mask(inp.q, inp.k, bsa.MaskPolicy(0.0, rho, g), layout=lay))
         .cpu().numpy() for rho in (0.75, 0.5)]
    assert ((r[0] > 0) & (r[0] <= r[1] + 1e-12) & (r[1] <= 1.0 + 1e-12)).all()


def test_config1_rows_vs_oracle(bsa):
    """N=8 VGGT frames (T=10,992), 2 heads: sampled q-blocks of the block map
    and the quadrant means against float64 from the same bf16 values."""
    from paper_2509_07120_b200.analysis import attention_quadrant_stats, block_attention_map

    c = dict(frames=8, patches=1369, specials=5, heads=2, d=64, seed=3)
    inp, lay = _inputs(bsa, c)
    q = inp.q.float().cpu().numpy().astype(np.float64)
    k = inp.k.float().cpu().numpy().astype(np.float64)
    scale = float(np.float32(oracle.head_scale(64)))
    perm, _ = oracle.partition_perm(8, 1369, 5)
    spec = np.zeros(lay.total_tokens, dtype=bool)
    spec[perm[:40]] = True
    pidx = oracle.patch_indices(8, 1369, 5)
    bm = block_attention_map(inp, lay).cpu().numpy()
    st = attention_quadrant_stats(inp, lay)
    sums = {quad: np.zeros(2) for quad in ("S2S", "S2P", "P2S", "P2P")}
    for h in range(2):
        for r0 in range(0, lay.total_tokens, 2048):
            s = (q[h, r0:r0 + 2048] @ k[h].T) * scale
            p = np.exp(s - s.max(axis=1, keepdims=True))
            p /= p.sum(axis=1, keepdims=True)
            rs = spec[r0:r0 + 2048]
            for quad, (qsel, ksel) in {"S2S": (rs, spec), "S2P": (rs, ~spec),
                                       "P2S": (~rs, spec), "P2P": (~rs, ~spec)}.items():
                sums[quad][h] += p[qsel][:, ksel].sum()
        for qb in (0, 37, 85):  # first, middle, ragged last patch q-block
            rows = pidx[qb * 128:(qb + 1) * 128]
            s = (q[h, rows] @ k[h].T) * scale
            p = np.exp(s - s.max(axis=1, keepdims=True))
            p /= p.sum(axis=1, keepdims=True)
            pk = p[:, pidx]
            ref = np.array([pk[:, b * 64:(b + 1) * 64].sum(axis=1).mean() for b in range(bm.shape[2])])
            np.testing.assert_allclose(bm[h, qb], ref, rtol=1e-3, atol=1e-7)
    ns, npch = 40, lay.total_tokens - 40
    count = {"S2S": ns * ns, "S2P": ns * npch, "P2S": npch * ns, "P2P": npch * npch}
    for quad in sums:
        np.testing.assert_allclose(st.means[quad], sums[quad] / count[quad], rtol=2e-4)


# ---- quadrant_stats on a materialised map: the reference's own tests
# (test_analysis.py:44-100) --------------------------------------------------

def _uniform_map(heads, n):
    return np.full((heads, n, n), 1.0 / n, dtype=np.float32)


def _flat_loop_oracle(attn_map, layout, bsa):
    h, n, _ = attn_map.shape
    spec = set(bsa.special_token_indices(layout).tolist())
    sums = {q: np.zeros(h) for q in ("S2S", "S2P", "P2S", "P2P")}
    counts = {q: 0 for q in sums}
    maxes = {q: np.full(h, -np.inf) for q in sums}
    for qi in range(n):
        for ki in range(n):
            quad = ("S" if qi in spec else "P") + "2" + ("S" if ki in spec else "P")
            counts[quad] += 1
            sums[quad] += attn_map[:, qi, ki]
            maxes[quad] = np.maximum(maxes[quad], attn_map[:, qi, ki])
    return ({q: sums[q] / counts[q] for q in sums if counts[q]},
            {q: maxes[q] for q in maxes if counts[q]}, counts)


def test_quadrant_stats_reference_cases(bsa):
    from paper_2509_07120_b200.analysis import quadrant_stats

    lay = bsa.TokenLayout(frames=2, patches_per_frame=6, specials_per_frame=2)
    n = lay.total_tokens
    st = quadrant_stats(_uniform_map(2, n), lay)
    for quad in ("S2S", "S2P", "P2S", "P2P"):
        np.testing.assert_allclose(st.means[quad], 1.0 / n, atol=1e-7)
        np.testing.assert_allclose(st.maxes[quad], 1.0 / n, atol=1e-7)
    lay0 = bsa.TokenLayout(frames=1, patches_per_frame=8, specials_per_frame=0)
    st0 = quadrant_stats(_uniform_map(1, 8), lay0)
    assert set(st0.means) == {"P2P"}
    rng = np.random.default_rng(0)
    lay2 = bsa.TokenLayout(frames=2, patches_per_frame=5, specials_per_frame=2)
    n2 = lay2.total_tokens
    m = np.exp(rng.standard_normal((2, n2, n2)).astype(np.float32))
    m /= m.sum(axis=2, keepdims=True)
    st2 = quadrant_stats(m, lay2)
    means, maxes, counts = _flat_loop_oracle(m, lay2, bsa)
    for quad in means:
        np.testing.assert_allclose(st2.means[quad], means[quad], atol=1e-6)
        np.testing.assert_allclose(st2.maxes[quad], maxes[quad], atol=1e-6)
    assert sum(counts.values()) == n2 * n2
    with pytest.raises(ValueError, match="sum"):
        quadrant_stats(np.ones((1, 4, 4), dtype=np.float32),
                       bsa.TokenLayout(frames=1, patches_per_frame=4, specials_per_frame=0))
    agg = quadrant_stats(_uniform_map(3, 4), bsa.TokenLayout(1, 4, 0)).aggregate()
    assert agg["P2P"][0] == pytest.approx(0.25) and agg["P2P"][1] == pytest.approx(0.0)
