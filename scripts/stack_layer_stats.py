"""Per-layer attention statistics of the config-3 stack (random init):
quadrant mean/max (the paper's attention-map analysis vs layer index) and the
predicted mask's recall of patch attention mass, as CSV. Streamed on the GPU
(analysis.py): no T x T map at any N."""
import argparse
import csv
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_07120_b200 as bsa  # noqa: E402
from paper_2509_07120_b200.stack import GlobalAttentionStack, policy_for  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--frames", type=int, default=50)
ap.add_argument("--layers", type=int, default=24)
ap.add_argument("--tau", type=float, default=0.0)
ap.add_argument("--rho", type=float, default=0.75)
ap.add_argument("--csv", default=None)
a = ap.parse_args()
lay = bsa.TokenLayout(a.frames, 1369, 5)
stack = GlobalAttentionStack(layers=a.layers)
g = torch.Generator(device="cuda").manual_seed(0)
x = torch.randn((lay.total_tokens, stack.dim), generator=g, device="cuda").to(torch.bfloat16)
t0 = time.time()
rows = stack.layer_statistics(x, lay, policy_for(lay, a.tau, a.rho))
torch.cuda.synchronize()
out = open(a.csv, "w", newline="") if a.csv else sys.stdout
w = csv.writer(out)
w.writerow(["layer", "quadrant", "mean_of_heads_mean", "mean_of_heads_max", "mask_recall"])
for r in rows:
    for quad in r["means"]:
        w.writerow([r["layer"], quad, f"{r['means'][quad].mean():.6g}",
                    f"{r['maxes'][quad].mean():.6g}", f"{r['recall']:.6g}"])
print(f"# {a.layers} layers at N={a.frames} in {time.time() - t0:.1f} s", file=sys.stderr)
