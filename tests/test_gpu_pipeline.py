"""Host-memory layer pipeline (pipeline.py): per-head-chunk H2D / kernels /
D2H on three streams must give exactly the device-resident result."""

import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("part", [True, False])
@pytest.mark.parametrize("chunk", [1, 2, 3, "auto", [2, 1, 2]])
def test_pipeline_equals_device_path(chunk, part):
    import torch
    import paper_2509_07120_b200 as bsa
    from paper_2509_07120_b200.pipeline import HostLayerPipeline

    lay = bsa.TokenLayout(3, 600, 5)
    H, T, d = 5, lay.total_tokens, 64
    g = torch.Generator().manual_seed(7)
    q, k, v = (torch.randn((H, T, d), generator=g).to(torch.bfloat16).pin_memory()
               for _ in range(3))
    pol = bsa.MaskPolicy(0.4, 0.8, bsa.BlockGeometry(lay.patch_tokens, 128, 64))
    pipe = HostLayerPipeline(H, T, d, torch.bfloat16, chunk_heads=chunk, partitioned_copies=part)
    out = pipe.run(q, k, v, lay, pol)
    out2 = pipe.run(q, k, v, lay, pol)  # buffers reused
    dq, dk, dv = (t.cuda() for t in (q, k, v))
    mask = bsa.predict_mask(dq, dk, pol, layout=lay)
    ref = bsa.sparse_attention(bsa.SparseAttentionJob(bsa.AttentionInputs(dq, dk, dv), lay, mask))
    assert out.device.type == "cpu"
    assert torch.equal(out, ref.cpu())
    assert torch.equal(out2, out)
    with pytest.raises(ValueError):
        pipe.run(dq, dk, dv, lay, pol)  # device tensors are refused


@pytest.mark.parametrize("specials_first", [True, False])
def test_copy_tokens_roundtrip(specials_first):
    """bsa_copy_tokens: interleaved host rows -> partitioned device rows is
    x[:, perm] (partition_permutation), and back is the identity."""
    import numpy as np
    import torch
    import paper_2509_07120_b200 as bsa
    from paper_2509_07120_b200 import _native as N
    lay = bsa.TokenLayout(4, 300, 3, specials_first=specials_first)
    H, T = 3, lay.total_tokens
    x = torch.randn((H, T, 64)).to(torch.bfloat16).pin_memory()
    dev = torch.empty((H, T, 64), dtype=torch.bfloat16, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    N.check(N.lib().bsa_copy_tokens(dev.data_ptr(), x.data_ptr(), N.layout_desc(lay), H, 128, 1, st),
            "copy_tokens")
    perm, _ = bsa.partition_permutation(lay)
    assert torch.equal(dev.cpu(), x[:, torch.from_numpy(perm)])
    back = torch.empty_like(x).pin_memory()
    N.check(N.lib().bsa_copy_tokens(back.data_ptr(), dev.data_ptr(), N.layout_desc(lay), H, 128, 0, st),
            "copy_tokens")
    torch.cuda.synchronize()
    assert torch.equal(back, x)
    assert np.array_equal(perm[: lay.special_tokens], bsa.special_token_indices(lay))
