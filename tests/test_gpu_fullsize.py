"""Parity at BASELINE.json's full sizes, through properties that do not need
the CPU to redo the whole layer:
* config-3 shape (the bench workload: N=200, 16 heads, tau=0, rho=0.75):
  every mask row keeps exactly k_floor blocks; masks nest in rho; head 0's
  mask is bit-exact against the C oracle at full size; sampled output rows
  (special and patch, first / middle / ragged-last q-blocks, two heads) match
  the float64 oracle within the bf16 tolerance; reruns are bit-identical;
* config-5 single-GPU leg (N=1000, 2 heads): row counts, sampled rows,
  determinism."""

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

BF16_REL_TOL = 2e-2


@pytest.fixture(scope="module")
def bsa():
    import paper_2509_07120_b200 as m
    return m


def _inputs(bsa, frames, heads, seed):
    import torch
    lay = bsa.TokenLayout(frames, 1369, 5)
    g = torch.Generator(device="cuda").manual_seed(seed)
    q, k, v = (torch.randn((heads, lay.total_tokens, 64), generator=g, device="cuda")
               .to(torch.bfloat16) for _ in range(3))
    return lay, q, k, v


def _sample_rows(lay, bq=128):
    """Source-order rows: specials of the first and last frame, and patch
    rows of the first, a middle and the (ragged) last q-block."""
    perm, _ = oracle.partition_perm(lay.frames, lay.patches_per_frame, lay.specials_per_frame)
    ns, tp = lay.special_tokens, lay.patch_tokens
    nq = -(-tp // bq)
    part = [0, ns - 1, ns, ns + 57, ns + (nq // 2) * bq + 3, ns + (nq - 1) * bq,
            ns + tp - 1]
    return sorted(set(int(perm[p]) for p in part))


def _check_rows(bsa, lay, q, k, v, mask, out, heads):
    rows = _sample_rows(lay)
    for h in heads:
        qh, kh, vh = (t[h:h + 1].float().cpu().numpy() for t in (q, k, v))
        ref = oracle.masked_attention_f64(qh, kh, vh, lay.frames, lay.patches_per_frame,
                                          lay.specials_per_frame, mask.blocks[h:h + 1], 128, 64,
                                          rows=rows)
        got = out[h:h + 1, rows].float().cpu().numpy()
        err = np.abs(got - ref).max() / np.abs(ref).max()
        assert err <= BF16_REL_TOL, f"head {h}: rel err {err}"


def test_bench_workload_n200(bsa):
    import torch
    lay, q, k, v = _inputs(bsa, 200, 16, 0)
    g = bsa.BlockGeometry(lay.patch_tokens, 128, 64)
    pol = bsa.MaskPolicy(0.0, 0.75, g)
    mask = bsa.predict_mask(q, k, pol, layout=lay)
    assert bool((mask.device_counts() == pol.min_blocks).all())
    tighter = bsa.predict_mask(q, k, bsa.MaskPolicy(0.0, 0.8, g), layout=lay)
    assert not bool((tighter.device_bits() & ~mask.device_bits()).any())
    # head 0 scoring bit-exact against the C restatement of numpy/OpenBLAS
    pidx = bsa.patch_token_indices(lay)
    qp, kp = (t[0:1, torch.from_numpy(pidx).cuda()].float().cpu().numpy() for t in (q, k))
    om, _ = oracle.predict_mask(qp, kp, 128, 64, 0.0, 0.75)
    assert np.array_equal(om[0], mask.blocks[0])
    job = bsa.SparseAttentionJob(bsa.AttentionInputs(q, k, v), lay, mask)
    out = bsa.sparse_attention(job)
    _check_rows(bsa, lay, q, k, v, mask, out, heads=(0, 15))
    assert torch.equal(bsa.sparse_attention(job), out)


def test_config5_single_gpu_leg_n1000(bsa):
    import torch
    lay, q, k, v = _inputs(bsa, 1000, 2, 1)
    g = bsa.BlockGeometry(lay.patch_tokens, 128, 64)
    pol = bsa.MaskPolicy(0.0, 0.5, g)
    mask = bsa.predict_mask(q, k, pol, layout=lay)
    assert bool((mask.device_counts() == pol.min_blocks).all())
    job = bsa.SparseAttentionJob(bsa.AttentionInputs(q, k, v), lay, mask)
    out = bsa.sparse_attention(job)
    _check_rows(bsa, lay, q, k, v, mask, out, heads=(1,))
    assert torch.equal(bsa.sparse_attention(job), out)


def test_cdf_policy_full_size_mask_exact(bsa):
    """tau > 0 (the CDF branch with the exact fixed-point mass search) at the
    bench size: head 3's whole mask bit-exact against the C oracle."""
    import torch
    lay, q, k, _ = _inputs(bsa, 200, 4, 2)
    g = bsa.BlockGeometry(lay.patch_tokens, 128, 64)
    pol = bsa.MaskPolicy(0.4, 0.8, g)
    mask = bsa.predict_mask(q, k, pol, layout=lay)
    assert bool((mask.device_counts() >= pol.min_blocks).all())
    pidx = torch.from_numpy(bsa.patch_token_indices(lay)).cuda()
    qp, kp = (t[3:4, pidx].float().cpu().numpy() for t in (q, k))
    om, oc = oracle.predict_mask(qp, kp, 128, 64, 0.4, 0.8)
    assert np.array_equal(om[0], mask.blocks[3])


def test_pi3_shape_n300(bsa):
    """Config 4: pi3-shaped layer, 4 register tokens per frame, N=300."""
    import torch
    lay = bsa.TokenLayout(300, 1369, 4)
    gen = torch.Generator(device="cuda").manual_seed(3)
    q, k, v = (torch.randn((2, lay.total_tokens, 64), generator=gen, device="cuda")
               .to(torch.bfloat16) for _ in range(3))
    g = bsa.BlockGeometry(lay.patch_tokens, 128, 64)
    pol = bsa.MaskPolicy(0.0, 0.75, g)
    mask = bsa.predict_mask(q, k, pol, layout=lay)
    assert bool((mask.device_counts() == pol.min_blocks).all())
    pidx = torch.from_numpy(bsa.patch_token_indices(lay)).cuda()
    qp, kp = (t[0:1, pidx].float().cpu().numpy() for t in (q, k))
    om, _ = oracle.predict_mask(qp, kp, 128, 64, 0.0, 0.75)
    assert np.array_equal(om[0], mask.blocks[0])
    out = bsa.sparse_attention(bsa.SparseAttentionJob(bsa.AttentionInputs(q, k, v), lay, mask))
    _check_rows(bsa, lay, q, k, v, mask, out, heads=(0,))


def test_host_pipeline_full_size_equals_device_path(bsa):
    """bench.py's e2e leg: the head-chunked host-memory pipeline at N=200, 16
    heads gives exactly the device-resident result."""
    import torch
    from paper_2509_07120_b200.pipeline import HostLayerPipeline
    lay, q, k, v = _inputs(bsa, 200, 16, 0)
    pol = bsa.MaskPolicy(0.0, 0.75, bsa.BlockGeometry(lay.patch_tokens, 128, 64))
    mask = bsa.predict_mask(q, k, pol, layout=lay)
    ref = bsa.sparse_attention(bsa.SparseAttentionJob(bsa.AttentionInputs(q, k, v), lay, mask))
    hq, hk, hv = (t.cpu().pin_memory() for t in (q, k, v))
    out = HostLayerPipeline(16, lay.total_tokens, 64).run(hq, hk, hv, lay, pol)
    assert torch.equal(out, ref.cpu())
