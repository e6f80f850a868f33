"""Host-memory layer pipeline (pipeline.py): per-head-chunk H2D / kernels /
D2H on three streams must give exactly the device-resident result."""

import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("chunk", [1, 2, 3, "auto", [2, 1, 2]])
def test_pipeline_equals_device_path(chunk):
    import torch
    import paper_2509_07120_b200 as bsa
    from paper_2509_07120_b200.pipeline import HostLayerPipeline

    lay = bsa.TokenLayout(3, 600, 5)
    H, T, d = 5, lay.total_tokens, 64
    g = torch.Generator().manual_seed(7)
    q, k, v = (torch.randn((H, T, d), generator=g).to(torch.bfloat16).pin_memory()
               for _ in range(3))
    pol = bsa.MaskPolicy(0.4, 0.8, bsa.BlockGeometry(lay.patch_tokens, 128, 64))
    pipe = HostLayerPipeline(H, T, d, torch.bfloat16, chunk_heads=chunk)
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
