"""The fused QKV projection: tcgen05 GEMM whose
epilogue writes head-major partitioned Q/K/V and the pooled patch Q/K.

Bars:
* Q/K/V: the fp32-accumulated product rounded once to bf16: every element
  within half a bf16 ulp of x W^T + b (float64, same bf16 inputs) plus the
  fp32 accumulation error 2^-21 |x||W|^T (cancellation); and > 99.9% of the
  elements equal to cuBLAS's F.linear on the same inputs;
* pooled Q/K: bit-identical to block_pool of the bf16 patch rows (the
  device pool kernel, itself bit-exact with the reference) and to the
  oracle's numpy block_pool (maskpred.py:104-120) on small cases;
* predict_mask_pooled: mask bits, counts and probabilities identical to
  predict_mask on the Q/K the means were pooled from.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def bsa():
    import paper_2509_07120_b200 as m
    return m


def _inputs(F, P, S, H, seed, bias=True):
    import torch
    from paper_2509_07120_b200 import TokenLayout
    lay = TokenLayout(F, P, S)
    C = H * 64
    g = torch.Generator(device="cpu").manual_seed(seed)
    x = torch.randn((lay.total_tokens, C), generator=g).to("cuda", torch.bfloat16)
    w = (torch.randn((3 * C, C), generator=g) / np.sqrt(C)).to("cuda", torch.bfloat16)
    b = (0.1 * torch.randn((3 * C,), generator=g)).to("cuda", torch.bfloat16) if bias else None
    return lay, x, w, b


def _ref_qkv(x, w, b, H):
    xd, wd = x.double(), w.double()
    y = xd @ wd.T
    if b is not None:
        y = y + b.double()
    T = x.shape[0]
    return y.view(T, 3, H, 64).permute(1, 2, 0, 3)  # (3, H, T, 64) float64


CASES = [
    # frames, patches, specials, heads: ragged last q/k blocks, partial special tile
    (3, 300, 5, 4),
    (2, 1369, 5, 4),     # VGGT frame size (blocks straddle frames)
    (4, 1369, 5, 16),    # headline head count, C = 1024
    (1, 70, 0, 4),       # no special rows, one ragged q-block
    (1, 129, 200, 4),    # more special rows than patches; 1-row last q-block
]


@pytest.mark.parametrize("F,P,S,H", CASES)
def test_qkv_projection_values_and_pools(bsa, F, P, S, H):
    import torch
    lay, x, w, b = _inputs(F, P, S, H, seed=F * 7 + P + S + H)
    q, k, v, qp, kp = bsa.qkv_projection(x, w, b, H, lay)
    torch.cuda.synchronize()
    ref = _ref_qkv(x, w, b, H)
    # |x| |W|^T: the scale of the fp32 accumulation error (cancellation cases)
    mag = _ref_qkv(x.abs(), w.abs(), None, H)
    T = lay.total_tokens
    cub = torch.nn.functional.linear(x, w, b).view(T, 3, H, 64).permute(1, 2, 0, 3)
    for i, (name, got) in enumerate((("q", q), ("k", k), ("v", v))):
        r = ref[i]
        err = (got.double() - r).abs()
        bound = r.abs() * 2.0 ** -8 + mag[i] * 2.0 ** -21  # final bf16 rounding + fp32 sums
        assert bool((err <= bound).all()), (
            f"{name}: {int((err > bound).sum())} elements beyond the bound, max err {err.max().item()}")
        same = (got == cub[i]).double().mean().item()
        assert same > 0.999, f"{name}: only {same:.5f} of elements equal cuBLAS's"
    Ts = lay.special_tokens
    g = bsa.geometry_for(lay)
    assert torch.equal(qp, bsa.block_pool(q[:, Ts:], 128)), "pooled Q differs from block_pool"
    assert torch.equal(kp, bsa.block_pool(k[:, Ts:], 64)), "pooled K differs from block_pool"
    assert qp.shape == (H, g.nq_blocks, 64) and kp.shape == (H, g.nk_blocks, 64)


def test_full_size_n200_pools_and_mask(bsa):
    """The config-3 layer shape (N=200, 16 heads, T=274,800), no bias: pools
    bit-identical to block_pool of the outputs, mask identical to
    predict_mask's, and Q/K/V equal to cuBLAS's projection (same rounding)."""
    import torch
    lay, x, w, _ = _inputs(200, 1369, 5, 16, seed=200, bias=False)
    q, k, v, qp, kp = bsa.qkv_projection(x, w, None, 16, lay)
    Ts = lay.special_tokens
    assert torch.equal(qp, bsa.block_pool(q[:, Ts:], 128, validate=False))
    assert torch.equal(kp, bsa.block_pool(k[:, Ts:], 64, validate=False))
    pol = bsa.MaskPolicy(0.0, 0.75, bsa.geometry_for(lay))
    m1 = bsa.predict_mask_pooled(qp, kp, pol)
    m2 = bsa.predict_mask(q[:, Ts:], k[:, Ts:], pol, validate=False)
    assert torch.equal(m1.device_bits(), m2.device_bits())
    T = lay.total_tokens
    cub = torch.nn.functional.linear(x, w).view(T, 3, 16, 64).permute(1, 2, 0, 3)
    for i, got in enumerate((q, k, v)):
        same = (got == cub[i]).double().mean().item()
        assert same > 0.999, same


def test_config5_size_n1000(bsa):
    """N=1000 frames (T=1,374,000; x is 2.8 GB, Q/K/V 8.4 GB): 64-bit
    offsets throughout; pools bit-identical to block_pool; values equal to
    cuBLAS's on a sample of rows spread over the whole sequence."""
    import torch
    lay, x, w, b = _inputs(1000, 1369, 5, 16, seed=1000)
    q, k, v, qp, kp = bsa.qkv_projection(x, w, b, 16, lay)
    Ts = lay.special_tokens
    assert torch.equal(qp, bsa.block_pool(q[:, Ts:], 128, validate=False))
    assert torch.equal(kp, bsa.block_pool(k[:, Ts:], 64, validate=False))
    rows = torch.linspace(0, lay.total_tokens - 1, 4096, device="cuda").long()
    cub = torch.nn.functional.linear(x[rows], w, b).view(-1, 3, 16, 64).permute(1, 2, 0, 3)
    for i, got in enumerate((q, k, v)):
        same = (got[:, rows] == cub[i]).double().mean().item()
        assert same > 0.999, same


def test_pools_match_oracle_numpy(bsa):
    import oracle
    lay, x, w, b = _inputs(3, 300, 5, 4, seed=11)
    q, k, _, qp, kp = bsa.qkv_projection(x, w, b, 4, lay)
    Ts = lay.special_tokens
    qn = q[:, Ts:].float().cpu().numpy()
    kn = k[:, Ts:].float().cpu().numpy()
    np.testing.assert_array_equal(qp.cpu().numpy(), oracle.block_pool(qn, 128))
    np.testing.assert_array_equal(kp.cpu().numpy(), oracle.block_pool(kn, 64))


@pytest.mark.parametrize("tau,rho", [(0.4, 0.8), (0.0, 0.75), (0.9, 0.5)])
def test_predict_mask_pooled_equals_predict_mask(bsa, tau, rho):
    import torch
    lay, x, w, b = _inputs(4, 1369, 5, 16, seed=3)
    q, k, _, qp, kp = bsa.qkv_projection(x, w, b, 16, lay)
    g = bsa.geometry_for(lay)
    pol = bsa.MaskPolicy(tau, rho, g)
    m1, p1 = bsa.predict_mask_pooled(qp, kp, pol, return_probs=True)
    Ts = lay.special_tokens  # q/k rows are in partitioned order: patches follow the specials
    m2, p2 = bsa.predict_mask(q[:, Ts:], k[:, Ts:], pol, return_probs=True)
    assert torch.equal(m1.device_bits(), m2.device_bits())
    assert torch.equal(m1.device_counts(), m2.device_counts())
    assert torch.equal(p1, p2)


def test_predict_mask_pooled_long_rows(bsa):
    """Long rows (N=500: 10,695 key blocks) run the one-row-per-CTA shape of
    the fused scoring kernel (16-CTA clusters); from the pools as well."""
    import torch
    lay = bsa.TokenLayout(500, 1369, 5)
    g = torch.Generator(device="cuda").manual_seed(9)
    q, k = (torch.randn((2, lay.total_tokens, 64), generator=g, device="cuda").to(torch.bfloat16)
            for _ in range(2))
    geo = bsa.geometry_for(lay)
    pol = bsa.MaskPolicy(0.4, 0.8, geo)
    pidx = torch.from_numpy(bsa.patch_token_indices(lay)).cuda()
    qp = bsa.block_pool(q[:, pidx].contiguous(), 128, validate=False)
    kp = bsa.block_pool(k[:, pidx].contiguous(), 64, validate=False)
    m1 = bsa.predict_mask_pooled(qp, kp, pol)
    m2 = bsa.predict_mask(q, k, pol, layout=lay)
    assert torch.equal(m1.device_bits(), m2.device_bits())
    assert torch.equal(m1.device_counts(), m2.device_counts())


def test_fused_layer_equals_composition(bsa):
    """The stack's fused attention branch is exactly qkv_projection ->
    predict_mask (on the full interleaved Q/K) -> sparse_attention."""
    import torch
    import torch.nn.functional as F
    from paper_2509_07120_b200.stack import GlobalAttentionStack, policy_for
    lay = bsa.TokenLayout(3, 1369, 5)
    st = GlobalAttentionStack(layers=1, heads=16, seed=5)
    pol = policy_for(lay, 0.0, 0.75)
    perm, _ = bsa.partition_permutation(lay)
    x = torch.randn((lay.total_tokens, 1024), generator=torch.Generator().manual_seed(1)).to(
        "cuda", torch.bfloat16)
    xp = x[torch.from_numpy(perm).cuda()]
    blk = st.blocks[0]
    got = st.attention_fused(xp, blk, lay, pol)
    h = F.layer_norm(xp, (1024,), blk.ln_w, blk.ln_b)
    q, k, v, _, _ = bsa.qkv_projection(h, blk.qkv_w, blk.qkv_b, 16, lay, pooled=False)
    Ts = lay.special_tokens
    mask = bsa.predict_mask(q[:, Ts:], k[:, Ts:], pol)
    o = bsa.sparse_attention(bsa.SparseAttentionJob(bsa.AttentionInputs(q, k, v), lay, mask),
                             inputs_permuted=True)
    want = F.linear(o.permute(1, 0, 2).reshape(lay.total_tokens, 1024), blk.proj_w, blk.proj_b)
    assert torch.equal(got, want)


def test_fused_stack_close_to_sparse_stack(bsa):
    """mode="fused" (own GEMM, pooled epilogue, permuted residual stream) vs
    mode="sparse" (cuBLAS projection, interleaved order): the projections
    round differently in the last bf16 bit, so the bar is the bf16 attention
    tolerance on the block output, not bit equality."""
    import torch
    from paper_2509_07120_b200.stack import GlobalAttentionStack, policy_for
    lay = bsa.TokenLayout(4, 1369, 5)
    st = GlobalAttentionStack(layers=2, heads=16, seed=2, mlp=True)
    pol = policy_for(lay, 0.0, 0.75)
    x = torch.randn((lay.total_tokens, 1024), generator=torch.Generator().manual_seed(4)).to(
        "cuda", torch.bfloat16)
    a = st.forward(x, lay, pol, mode="fused").float()
    r = st.forward(x, lay, pol, mode="sparse").float()
    rel = ((a - r).norm() / r.norm()).item()
    assert rel < 2e-2, rel


@pytest.mark.parametrize("S,specials_first", [(4, True), (5, False)])
def test_fused_stack_other_layouts(bsa, S, specials_first):
    """pi3-style 4 register tokens, and specials after the patches: the
    fused stack (partitioned residual stream) still matches the sparse
    stack within the bf16 tolerance."""
    import torch
    from paper_2509_07120_b200.stack import GlobalAttentionStack, policy_for
    lay = bsa.TokenLayout(3, 1369, S, specials_first=specials_first)
    st = GlobalAttentionStack(layers=2, heads=16, seed=3)
    pol = policy_for(lay, 0.0, 0.75)
    x = torch.randn((lay.total_tokens, 1024), generator=torch.Generator().manual_seed(8)).to(
        "cuda", torch.bfloat16)
    a = st.forward(x, lay, pol, mode="fused").float()
    r = st.forward(x, lay, pol, mode="sparse").float()
    assert ((a - r).norm() / r.norm()).item() < 2e-2


def test_qkv_projection_rejects_bad_inputs(bsa):
    import torch
    lay, x, w, b = _inputs(1, 70, 0, 4, seed=0)
    with pytest.raises(ValueError):
        bsa.qkv_projection(x.float(), w, b, 4, lay)
    with pytest.raises(ValueError):
        bsa.qkv_projection(x, w[:-1], b, 4, lay)
    with pytest.raises(ValueError):
        bsa.qkv_projection(x, w, b, 2, lay)
    with pytest.raises(ValueError):
        bsa.qkv_projection(x[:-1], w, b, 4, lay)
    with pytest.raises(ValueError):  # geometry other than 128/64
        bsa.qkv_projection(x, w, b, 4, lay, bsa.BlockGeometry(lay.patch_tokens, 64, 64))
    with pytest.raises(ValueError):
        bsa.predict_mask_pooled(torch.zeros(4, 3, 64, device="cuda"),
                                torch.zeros(4, 2, 64, device="cuda"),
                                bsa.MaskPolicy(0.0, 0.5, bsa.geometry_for(lay)))


# ---------------------------------------------------------------------------
# the output projection with its residual (qkv.proj_residual)
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("H,T,bias", [(4, 300, True), (16, 5496, True), (16, 27480, False),
                                      (4, 1, True), (8, 129, False)])
def test_proj_residual_values(bsa, H, T, bias):
    """out = residual + o' W^T + b with o' the token-major view of the
    head-major o: within half a bf16 ulp of float64 plus the fp32
    accumulation bound (one rounding of the whole sum), and within the
    rounding of torch's two-step residual + F.linear."""
    import torch
    C = H * 64
    g = torch.Generator(device="cpu").manual_seed(H * 1000 + T)
    o = torch.randn((H, T, 64), generator=g).to("cuda", torch.bfloat16)
    w = (torch.randn((C, C), generator=g) / np.sqrt(C)).to("cuda", torch.bfloat16)
    b = (0.1 * torch.randn((C,), generator=g)).to("cuda", torch.bfloat16) if bias else None
    res = torch.randn((T, C), generator=g).to("cuda", torch.bfloat16)
    out = bsa.proj_residual(o, w, b, res)
    ot = o.permute(1, 0, 2).reshape(T, C)
    ref = res.double() + ot.double() @ w.double().T + (b.double() if bias else 0.0)
    mag = res.double().abs() + ot.double().abs() @ w.double().abs().T
    err = (out.double() - ref).abs()
    bound = ref.abs() * 2.0 ** -8 + mag * 2.0 ** -21
    assert bool((err <= bound).all()), f"{int((err > bound).sum())} beyond bound, max {err.max().item()}"
    # torch rounds the projection y to bf16 before adding the residual:
    # its result is within half an ulp of |y| (plus its own final rounding)
    y = torch.nn.functional.linear(ot, w, b)
    tref = (res + y).double()
    tb = (tref.abs() + y.double().abs()) * 2.0 ** -8 + ref.abs() * 2.0 ** -8 + mag * 2.0 ** -20
    assert bool(((out.double() - tref).abs() <= tb).all())


def test_proj_residual_in_place_and_guards(bsa):
    import torch
    H, T = 4, 1000
    C = H * 64
    o = torch.randn((H, T, 64), device="cuda").to(torch.bfloat16)
    w = (torch.randn((C, C), device="cuda") / 16).to(torch.bfloat16)
    res = torch.randn((T, C), device="cuda").to(torch.bfloat16)
    want = bsa.proj_residual(o, w, None, res)
    x = res.clone()
    got = bsa.proj_residual(o, w, None, x, out=x)
    assert got.data_ptr() == x.data_ptr() and torch.equal(got, want)
    with pytest.raises(ValueError):
        bsa.proj_residual(o.float(), w, None, res)
    with pytest.raises(ValueError):
        bsa.proj_residual(o, w[:, :-1], None, res)
    with pytest.raises(ValueError):
        bsa.proj_residual(o, w, None, res[:-1])
    with pytest.raises(ValueError):  # C % 256 != 0
        o2 = torch.zeros((2, T, 64), device="cuda", dtype=torch.bfloat16)
        bsa.proj_residual(o2, torch.zeros((128, 128), device="cuda", dtype=torch.bfloat16), None,
                          torch.zeros((T, 128), device="cuda", dtype=torch.bfloat16))
