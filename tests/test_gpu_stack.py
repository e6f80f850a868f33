"""The config-3 model harness (paper_2509_07120_b200/stack.py) on the B200:
with every key block selected the sparse stack equals the dense one."""

import pytest

pytestmark = pytest.mark.gpu


def test_stack_full_mask_matches_dense():
    import torch
    from paper_2509_07120_b200 import TokenLayout
    from paper_2509_07120_b200.stack import GlobalAttentionStack, policy_for

    lay = TokenLayout(3, 700, 5)
    stack = GlobalAttentionStack(layers=2, seed=1, mlp=True)
    g = torch.Generator(device="cuda").manual_seed(3)
    x = torch.randn((lay.total_tokens, stack.dim), generator=g, device="cuda").to(torch.bfloat16)
    pol = policy_for(lay, 0.0, 0.0)  # rho = 0: every block kept
    ys = stack(x, lay, pol, "sparse").float()
    yd = stack(x, lay, None, "dense").float()
    rel = float((ys - yd).abs().max() / yd.abs().max())
    assert rel <= 2e-2, rel


def test_stack_sparse_runs_and_validates():
    import torch
    from paper_2509_07120_b200 import TokenLayout
    from paper_2509_07120_b200.stack import GlobalAttentionStack, policy_for

    lay = TokenLayout(4, 1369, 4)  # pi3-style: 4 register tokens per frame
    stack = GlobalAttentionStack(layers=2)
    x = torch.randn((lay.total_tokens, stack.dim), device="cuda").to(torch.bfloat16)
    y = stack(x, lay, policy_for(lay, 0.4, 0.8), "sparse")
    assert torch.isfinite(y).all()
    with pytest.raises(ValueError):
        stack(x[:-1], lay, policy_for(lay, 0.4, 0.8), "sparse")
    with pytest.raises(ValueError):
        stack(x, lay, None, "sparse")


def test_layer_statistics_match_materialised_maps():
    """Per-layer streamed quadrant stats equal quadrant_stats of the dense
    map of the same layer's q/k (small N, 3 layers)."""
    import numpy as np
    import torch
    import torch.nn.functional as F
    import paper_2509_07120_b200 as bsa
    from paper_2509_07120_b200.analysis import quadrant_stats
    from paper_2509_07120_b200.stack import GlobalAttentionStack, policy_for

    lay = bsa.TokenLayout(2, 300, 5)
    st = GlobalAttentionStack(layers=3, seed=1)
    g = torch.Generator(device="cuda").manual_seed(2)
    x = torch.randn((lay.total_tokens, st.dim), generator=g, device="cuda").to(torch.bfloat16)
    rows = st.layer_statistics(x, lay, policy_for(lay, 0.0, 0.75), mode="dense")
    assert [r["layer"] for r in rows] == [0, 1, 2]
    T, C = x.shape
    for r, blk in zip(rows, st.blocks):
        h = F.layer_norm(x, (C,), blk.ln_w, blk.ln_b)
        qkv = F.linear(h, blk.qkv_w, blk.qkv_b).view(T, 3, 16, 64).permute(1, 2, 0, 3)
        s = torch.matmul(qkv[0].float(), qkv[1].float().transpose(1, 2)) * 0.125
        ref = quadrant_stats(torch.softmax(s.double(), dim=-1).float(), lay)
        for quad in ref.means:
            np.testing.assert_allclose(r["means"][quad], ref.means[quad], rtol=2e-3)
            np.testing.assert_allclose(r["maxes"][quad], ref.maxes[quad], rtol=2e-3)
        assert 0.0 < r["recall"] <= 1.0
        x = x + st.attention(x, blk, lay, None, "dense")


def test_stack_forward_sharded_world1_equals_forward():
    """Config 3's multi-GPU form (frames split over the ranks) through a real
    NCCL group of one rank: bit-identical to the single-GPU stack, for the
    scatter (persistent IPC target) and reduce-scatter combines."""
    import os
    import socket

    import torch
    import torch.distributed as dist
    from paper_2509_07120_b200 import TokenLayout
    from paper_2509_07120_b200.stack import GlobalAttentionStack, policy_for

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        lay = TokenLayout(3, 700, 5)
        stack = GlobalAttentionStack(layers=3, seed=2, mlp=True)
        g = torch.Generator(device="cuda").manual_seed(5)
        x = torch.randn((lay.total_tokens, stack.dim), generator=g, device="cuda").to(torch.bfloat16)
        pol = policy_for(lay, 0.4, 0.8)
        ref = stack(x, lay, pol, "sparse")
        for combine, chunk in (("auto", None), ("reduce_scatter", 4), ("allreduce", None)):
            y = stack.forward_sharded(x, lay, pol, combine=combine, chunk_heads=chunk)
            assert torch.equal(y, ref), combine
        with pytest.raises(ValueError):
            stack.forward_sharded(x[:-1], lay, pol)
    finally:
        dist.destroy_process_group()
