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


def _row_rel(got, ref):
    """max over rows of ||o - ref|| / ||ref||: a row with small outputs cannot
    hide behind the tensor's global max."""
    num = np.linalg.norm((got - ref).reshape(-1, got.shape[-1]), axis=1)
    den = np.linalg.norm(ref.reshape(-1, ref.shape[-1]), axis=1)
    return float((num / np.maximum(den, 1e-30)).max())


def _check_rows(bsa, lay, q, k, v, mask, out, heads, rows=None):
    rows = _sample_rows(lay) if rows is None else rows
    for h in heads:
        qh, kh, vh = (t[h:h + 1].float().cpu().numpy() for t in (q, k, v))
        ref = oracle.masked_attention_f64(qh, kh, vh, lay.frames, lay.patches_per_frame,
                                          lay.specials_per_frame, mask.blocks[h:h + 1], 128, 64,
                                          rows=rows)
        got = out[h:h + 1, rows].float().cpu().numpy()
        err = np.abs(got - ref).max() / np.abs(ref).max()
        assert err <= BF16_REL_TOL, f"head {h}: rel err {err}"
        assert _row_rel(got, ref) <= BF16_REL_TOL, f"head {h}: per-row rel err"


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


def _sha(a):
    import hashlib
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.mark.parametrize("name", ["n200h2", "n200h2_bf16"])
def test_headline_masks_match_reference_fixture(bsa, name):
    """N=200 frames (the headline size), 2 heads: pooled Q/K, probabilities
    and masks for tau=0/rho=0.75 and tau=0.4/rho=0.8 equal the REFERENCE's
    own (tests/golden/make_golden.py ran bsattn.predict_mask at this size;
    maskpred.py:104-194), digest for digest; fp32 inputs and bf16 inputs."""
    import os

    import torch
    from golden_inputs import FULL_POLICIES, bf16_round, make_qkv

    z = np.load(os.path.join(os.path.dirname(__file__), "golden", f"full_{name}.npz"))
    lay = bsa.TokenLayout(int(z["frames"]), int(z["patches"]), int(z["specials"]))
    q, k, _ = make_qkv(int(z["heads"]), lay.total_tokens, int(z["d"]), int(z["seed"]))
    dt = torch.float32
    if bool(z["bf16"]):
        q, k, dt = bf16_round(q), bf16_round(k), torch.bfloat16
    qd, kd = (torch.from_numpy(x).to("cuda", dt) for x in (q, k))
    g = bsa.BlockGeometry(lay.patch_tokens, 128, 64)
    pidx = torch.from_numpy(bsa.patch_token_indices(lay)).cuda()
    assert _sha(bsa.block_pool(qd[:, pidx], 128).cpu().numpy()) == str(z["qp_sha"])
    assert _sha(bsa.block_pool(kd[:, pidx], 64).cpu().numpy()) == str(z["kp_sha"])
    for i, (tau, rho) in enumerate(FULL_POLICIES):
        mask, probs = bsa.predict_mask(qd, kd, bsa.MaskPolicy(tau, rho, g), layout=lay,
                                       return_probs=True)
        if i == 0:
            assert _sha(probs.cpu().numpy()) == str(z["probs_sha"])
        assert np.array_equal(mask.device_counts().cpu().numpy().reshape(z[f"mask{i}_counts"].shape),
                              z[f"mask{i}_counts"])
        assert _sha(mask.device_bits().cpu().numpy()) == str(z[f"mask{i}_sha"]), (tau, rho)


def test_bench_workload_all_heads(bsa):
    """The bench workload itself (N=200, 16 heads, tau=0, rho=0.75, bf16):
    all 16 heads' masks bit-exact against the C restatement; per head one
    whole q-block (128 rows) and, for heads 0 and 1, all 1000 special rows
    against the float64 oracle, per row and globally."""
    import torch
    lay, q, k, v = _inputs(bsa, 200, 16, 0)
    g = bsa.BlockGeometry(lay.patch_tokens, 128, 64)
    mask = bsa.predict_mask(q, k, bsa.MaskPolicy(0.0, 0.75, g), layout=lay)
    pidx = torch.from_numpy(bsa.patch_token_indices(lay)).cuda()
    qp, kp = (t[:, pidx].float().cpu().numpy() for t in (q, k))
    om, _ = oracle.predict_mask(qp, kp, 128, 64, 0.0, 0.75)
    assert np.array_equal(om, mask.blocks), "N=200 16-head mask differs from the oracle"
    out = bsa.sparse_attention(bsa.SparseAttentionJob(bsa.AttentionInputs(q, k, v), lay, mask))
    perm, _ = oracle.partition_perm(lay.frames, lay.patches_per_frame, lay.specials_per_frame)
    ns = lay.special_tokens
    rng = np.random.default_rng(0)
    for h in range(16):
        qb = int(rng.integers(g.nq_blocks))
        part = list(range(ns + qb * 128, ns + min((qb + 1) * 128, lay.patch_tokens)))
        if h < 2:
            part += list(range(ns))
        _check_rows(bsa, lay, q, k, v, mask, out, heads=(h,),
                    rows=sorted(int(perm[p]) for p in part))
