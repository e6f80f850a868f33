"""Dense attention-map statistics, CPU side: the
float64 oracle restatement against fixtures the REFERENCE produced
(dense_attention_map + quadrant_stats, tests/golden/make_golden.py), and the
quadrant reduction from row statistics (analysis.quadrant_stats_from_rows)
against the oracle on row statistics computed here in float64."""

import os

import numpy as np
import pytest
import torch

import oracle
from golden_inputs import CASES_MAP, bf16_round, make_qkv

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _case(c):
    g = np.load(os.path.join(GOLDEN, f"{c['name']}.npz"))
    q, k, _ = make_qkv(c["heads"], c["frames"] * (c["patches"] + c["specials"]), c["d"], c["seed"])
    return g, bf16_round(q), bf16_round(k)


@pytest.mark.parametrize("c", CASES_MAP, ids=[c["name"] for c in CASES_MAP])
def test_oracle_matches_reference_fixture(c):
    g, q, k = _case(c)
    p = oracle.attention_map_f64(q, k)
    means, maxes = oracle.quadrant_stats_f64(p, c["frames"], c["patches"], c["specials"])
    assert sorted(means) == sorted(str(x) for x in g["quads"])
    for quad in means:
        np.testing.assert_allclose(means[quad], g[f"mean_{quad}"], rtol=1e-5)
        np.testing.assert_allclose(maxes[quad], g[f"max_{quad}"], rtol=1e-5)
    bm = oracle.block_attention_map_f64(p, c["frames"], c["patches"], c["specials"])
    np.testing.assert_allclose(bm, g["block_map"], rtol=1e-4, atol=1e-7)


def _row_stats_f64(q, k):
    """The quantities bsa_attention_row_stats returns, in float64 (x = s*scale*log2 e)."""
    scale = float(np.float32(oracle.head_scale(q.shape[2])))
    x = np.einsum("htd,hsd->hts", q.astype(np.float64), k.astype(np.float64)) * scale / np.log(2)
    return x


@pytest.mark.parametrize("c", CASES_MAP, ids=[c["name"] for c in CASES_MAP])
def test_quadrant_reduction_from_row_stats(c):
    from paper_2509_07120_b200.analysis import quadrant_stats_from_rows
    from paper_2509_07120_b200.layout import TokenLayout

    g, q, k = _case(c)
    lay = TokenLayout(c["frames"], c["patches"], c["specials"])
    x = _row_stats_f64(q, k)
    perm, _ = oracle.partition_perm(c["frames"], c["patches"], c["specials"])
    spec = np.zeros(x.shape[2], dtype=bool)
    spec[perm[:c["frames"] * c["specials"]]] = True
    m = x.max(axis=2)
    e = np.exp2(x - m[..., None])
    neg = np.full_like(m, -np.inf)
    rs = np.stack([m, e[..., spec].sum(axis=2), e[..., ~spec].sum(axis=2),
                   x[..., spec].max(axis=2) if spec.any() else neg,
                   x[..., ~spec].max(axis=2)], axis=-1)
    st = quadrant_stats_from_rows(torch.from_numpy(rs), lay)
    assert sorted(st.means) == sorted(str(x) for x in g["quads"])
    for quad in st.means:
        np.testing.assert_allclose(st.means[quad], g[f"mean_{quad}"], rtol=1e-5)
        np.testing.assert_allclose(st.maxes[quad], g[f"max_{quad}"], rtol=1e-5)
    agg = st.aggregate()
    assert set(agg) == set(st.means)
