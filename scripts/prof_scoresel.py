"""predict_mask at the bench workload (N=200, 16 heads, bf16, tau=0 rho=0.75),
a few warm calls: the target of ncu captures of the scoring kernels."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_07120_b200 as bsa  # noqa: E402

F = int(os.environ.get("FRAMES", "200"))
lay = bsa.TokenLayout(F, 1369, 5)
g = bsa.BlockGeometry(lay.patch_tokens, 128, 64)
pol = bsa.MaskPolicy(float(os.environ.get("TAU", "0")), float(os.environ.get("RHO", "0.75")), g)
gen = torch.Generator(device="cuda")
gen.manual_seed(0)
q, k = (torch.randn((16, lay.total_tokens, 64), generator=gen, device="cuda").to(torch.bfloat16)
        for _ in range(2))
for _ in range(3):
    bsa.predict_mask(q, k, pol, layout=lay)
torch.cuda.synchronize()
