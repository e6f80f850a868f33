"""Argument guards of the public operators: the kernels
write through raw pointers, so every buffer the caller hands in is checked
before a launch; non-finite inputs are rejected like the reference's as_f32
(/root/reference/pkg/src/bsattn/tensorio.py:47-59); mixed dtypes promote
to fp32 like the reference."""

import numpy as np
import pytest

from golden_inputs import make_qkv

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def bsa():
    import paper_2509_07120_b200 as m
    return m


def _job(bsa, dtype=None):
    import torch
    lay = bsa.TokenLayout(2, 300, 5)
    q, k, v = (torch.from_numpy(x).cuda() for x in make_qkv(2, lay.total_tokens, 64, 5))
    if dtype is not None:
        q, k, v = (t.to(dtype) for t in (q, k, v))
    g = bsa.BlockGeometry(lay.patch_tokens, 128, 64)
    mask = bsa.predict_mask(q, k, bsa.MaskPolicy(0.0, 0.5, g), layout=lay)
    return bsa.SparseAttentionJob(bsa.AttentionInputs(q, k, v), lay, mask), q


def test_out_buffer_checked(bsa):
    import torch
    job, q = _job(bsa, torch.bfloat16)
    ref = bsa.sparse_attention(job)
    bad = [
        torch.empty((2, q.shape[1] - 1, 64), dtype=torch.bfloat16, device="cuda"),   # too small
        torch.empty((2, q.shape[1], 64), dtype=torch.float16, device="cuda"),        # dtype
        torch.empty((2, q.shape[1], 64), dtype=torch.float64, device="cuda"),
        torch.empty((2, 64, q.shape[1]), dtype=torch.bfloat16, device="cuda").transpose(1, 2),
        torch.empty((2, q.shape[1], 64), dtype=torch.bfloat16),                       # host
    ]
    for out in bad:
        with pytest.raises(ValueError):
            bsa.sparse_attention(job, out=out)
    out = torch.empty_like(ref)
    with pytest.raises(ValueError, match="conflicts"):
        bsa.sparse_attention(job, out=out, out_dtype=torch.float32)
    with pytest.raises(ValueError):
        bsa.sparse_attention(job, out_dtype=torch.float16)
    res = bsa.sparse_attention(job, out=out)
    assert res.data_ptr() == out.data_ptr()
    assert torch.equal(out, ref)
    o32 = torch.empty(ref.shape, dtype=torch.float32, device="cuda")
    bsa.sparse_attention(job, out=o32)
    assert float((o32 - ref.float()).abs().max()) < 1e-2


def test_non_finite_device_inputs_rejected(bsa):
    import torch
    lay = bsa.TokenLayout(1, 256, 0)
    q, k, v = (torch.from_numpy(x).cuda() for x in make_qkv(1, 256, 64, 3))
    g = bsa.BlockGeometry(256, 128, 64)
    pol = bsa.MaskPolicy(0.0, 0.5, g)
    for bad in (float("nan"), float("inf"), -float("inf")):
        kk = k.clone()
        kk[0, 17, 3] = bad
        with pytest.raises(ValueError, match="non-finite"):
            bsa.predict_mask(q, kk, pol)
        with pytest.raises(ValueError, match="non-finite"):
            bsa.AttentionInputs(q, kk, v)
        with pytest.raises(ValueError, match="non-finite"):
            bsa.AttentionInputs(q, k, kk.to(torch.bfloat16).float())
    # validate=False is the documented opt-out for pre-validated callers
    kk = k.clone()
    kk[0, 17, 3] = float("nan")
    bsa.predict_mask(q, kk, pol, validate=False)
    bsa.AttentionInputs(q, kk, v, validate=False)


def test_mixed_dtypes_promote_to_fp32(bsa):
    import torch
    lay = bsa.TokenLayout(1, 512, 0)
    q, k, v = (torch.from_numpy(x).cuda() for x in make_qkv(2, 512, 64, 4))
    g = bsa.BlockGeometry(512, 128, 64)
    pol = bsa.MaskPolicy(0.4, 0.8, g)
    qb = q.to(torch.bfloat16)
    # the reference sees both as fp32: bf16 q upcast exactly, k untouched
    want = bsa.predict_mask(qb.float(), k, pol).blocks
    got = bsa.predict_mask(qb, k, pol).blocks
    assert np.array_equal(got, want)
    inp = bsa.AttentionInputs(qb, k, v.to(torch.bfloat16))
    assert inp.q.dtype == inp.k.dtype == inp.v.dtype == torch.float32


def test_scatter_target_must_match_call(bsa):
    import torch
    from paper_2509_07120_b200.shard import ScatterTarget, ShardPlan, sharded_sparse_attention
    lay = bsa.TokenLayout(2, 300, 5)
    other = bsa.TokenLayout(2, 320, 5)
    q, k, v = (torch.from_numpy(x).cuda().to(torch.bfloat16)
               for x in make_qkv(2, lay.total_tokens, 64, 6))
    pol = bsa.MaskPolicy(0.0, 0.5, bsa.BlockGeometry(lay.patch_tokens, 128, 64))
    for tgt_lay, heads in ((lay, 3), (other, 2)):
        tgt = ScatterTarget(ShardPlan(tgt_lay, 1), heads, 64, 0, None, "cuda")
        with pytest.raises(ValueError, match="scatter_target"):
            sharded_sparse_attention(q, k, v, lay, pol, combine="scatter", scatter_target=tgt)
        tgt.close()
    tgt = ScatterTarget(ShardPlan(lay, 1), 2, 64, 0, None, "cuda")
    out = sharded_sparse_attention(q, k, v, lay, pol, combine="scatter", scatter_target=tgt)
    mask = bsa.predict_mask(q, k, pol, layout=lay)
    ref = bsa.sparse_attention(bsa.SparseAttentionJob(bsa.AttentionInputs(q, k, v), lay, mask))
    assert torch.equal(out, ref)
    tgt.close()
    with pytest.raises(ValueError, match="closed"):
        sharded_sparse_attention(q, k, v, lay, pol, combine="scatter", scatter_target=tgt)


def test_launch_follows_tensor_device(bsa):
    """Operators make the tensors' device current for the launch; with one
    GPU this checks the guard is a no-op that keeps results identical."""
    import torch
    job, q = _job(bsa, torch.bfloat16)
    with torch.cuda.device(0):
        a = bsa.sparse_attention(job)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        b = bsa.sparse_attention(job)
    s.synchronize()
    assert torch.equal(a, b)
    m = job.mask
    assert m.device_bits(q.device).device == q.device
    assert m.device_counts(q.device).device == q.device
