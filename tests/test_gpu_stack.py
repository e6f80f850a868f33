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
