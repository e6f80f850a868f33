"""One warm-up step + N profiled steps of the bench workload (for ncu)."""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_07120_b200 as bsa  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--frames", type=int, default=200)
ap.add_argument("--steps", type=int, default=1)
ap.add_argument("--tau", type=float, default=0.0)
ap.add_argument("--rho", type=float, default=0.75)
a = ap.parse_args()
lay = bsa.TokenLayout(a.frames, 1369, 5)
g = bsa.BlockGeometry(lay.patch_tokens, 128, 64)
pol = bsa.MaskPolicy(a.tau, a.rho, g)
gen = torch.Generator(device="cuda")
gen.manual_seed(0)
q, k, v = (torch.randn((16, lay.total_tokens, 64), generator=gen, device="cuda").to(torch.bfloat16)
           for _ in range(3))
for _ in range(1 + a.steps):
    mask = bsa.predict_mask(q, k, pol, layout=lay)
    out = bsa.sparse_attention(bsa.SparseAttentionJob(bsa.AttentionInputs(q, k, v), lay, mask))
torch.cuda.synchronize()
print("done")
