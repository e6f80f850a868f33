"""The fused scoring kernel (csrc/bsa_scoresel.cu) against the three-kernel
path it replaces on predict_mask (scores_kernel + softsel_kernel +
fallback_kernel), which the golden-fixture tests pin to the reference.

Bar: bit-identical masks, per-row counts and probabilities.  The path is
chosen once per process (BSA_SCORESEL, read at the first call), so each arm
runs in its own subprocess.  Cases cover the launch shapes (two CTAs of 4
rows per SM up to N ~ 230 frames, one CTA per SM beyond; the one-CTA shapes
also forced at every size via BSA_SCORESEL_SHAPE=1), bf16 and fp32 inputs,
the top-k floor and the CDF branch, rho 0 / 1, tau 1, head_dim 32, the shape
the fused kernel declines (head_dim 16) and rows handed to the exact
fallback (constant scores: every probability equal).
"""

import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CASES = [
    # name, frames, patches, specials, heads, d, dtype, tau, rho, seed, const
    ("n200_bf16", 200, 1369, 5, 2, 64, "bf16", 0.0, 0.75, 0, False),
    ("n200_cdf", 200, 1369, 5, 2, 64, "bf16", 0.4, 0.8, 1, False),
    ("n300_f32", 300, 1369, 4, 1, 64, "f32", 0.9, 0.5, 2, False),
    ("n8_f32", 8, 1369, 5, 16, 64, "f32", 0.0, 0.75, 3, False),
    ("n8_cdf", 8, 1369, 5, 16, 64, "f32", 0.5, 0.3, 4, False),
    ("n30_d32", 30, 1369, 5, 3, 32, "f32", 0.3, 0.6, 5, False),
    ("n3_d16", 3, 100, 2, 2, 16, "f32", 0.0, 0.5, 6, False),
    ("n50_rho0", 50, 1369, 5, 2, 64, "bf16", 0.2, 0.0, 7, False),
    ("n50_rho1", 50, 1369, 5, 2, 64, "bf16", 0.0, 1.0, 8, False),
    ("n50_tau1", 50, 1369, 5, 2, 64, "f32", 1.0, 0.9, 9, False),
    ("n20_const", 20, 1369, 5, 2, 64, "f32", 0.5, 0.6, 10, True),
]

ARM = r"""
import sys, numpy as np, torch
sys.path.insert(0, {root!r})
import paper_2509_07120_b200 as bsa
out = {{}}
for name, F, P, S, H, d, dt, tau, rho, seed, const in {cases!r}:
    lay = bsa.TokenLayout(F, P, S)
    g = bsa.BlockGeometry(lay.patch_tokens, 128, 64)
    pol = bsa.MaskPolicy(tau, rho, g)
    gen = torch.Generator(device="cuda"); gen.manual_seed(seed)
    dtype = torch.bfloat16 if dt == "bf16" else torch.float32
    q, k = (torch.randn((H, lay.total_tokens, d), generator=gen, device="cuda").to(dtype)
            for _ in range(2))
    if const:
        k = torch.ones_like(k)
    mask, probs = bsa.predict_mask(q, k, pol, layout=lay, return_probs=True)
    out[name + "/bits"] = mask.device_bits().cpu().numpy()
    out[name + "/counts"] = mask.device_counts().cpu().numpy()
    out[name + "/probs"] = probs.cpu().numpy().view(np.uint32)
np.savez({path!r}, **out)
"""


def _run(tmp_path, fused, shape="0"):
    path = str(tmp_path / f"arm{int(fused)}_{shape}.npz")
    code = ARM.format(root=ROOT, cases=CASES, path=path)
    env = dict(os.environ, BSA_SCORESEL="1" if fused else "0", BSA_SCORESEL_SHAPE=shape)
    subprocess.run([sys.executable, "-c", code], check=True, env=env, timeout=600)
    return np.load(path)


@pytest.mark.parametrize("shape", ["0", "1"])
def test_fused_scoring_bit_identical_to_three_kernel_path(tmp_path, shape):
    legacy, fused = _run(tmp_path, False), _run(tmp_path, True, shape)
    for name, *_ in CASES:
        for part in ("bits", "counts", "probs"):
            a, b = legacy[f"{name}/{part}"], fused[f"{name}/{part}"]
            assert a.shape == b.shape and np.array_equal(a, b), f"{name}: {part} differ"


def test_fused_scoring_engaged_at_the_bench_shape():
    """The C ABI reports the fused kernel's rows per CTA (0: three-kernel path)."""
    from paper_2509_07120_b200 import _native as N
    L = N.lib()
    assert L.bsa_scoring_rows_per_cta(4280, 64) == 4    # N=200 (bench): two CTAs per SM
    assert L.bsa_scoring_rows_per_cta(6418, 64) == 4    # N=300 (pi3)
    assert L.bsa_scoring_rows_per_cta(21390, 64) == 1   # N=1000: one row per CTA, 16-CTA clusters
    assert L.bsa_scoring_rows_per_cta(4280, 16) == 0    # head_dim not a multiple of 32
