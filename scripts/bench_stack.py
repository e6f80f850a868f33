"""BASELINE.json config 3: the 24-layer VGGT global-attention stack,
random-init weights, N frames, block-sparse vs dense (cuDNN SDPA) attention.
Prints one JSON line: ms per forward, per layer, split GEMM vs attention."""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_07120_b200 import TokenLayout  # noqa: E402
from paper_2509_07120_b200.stack import GlobalAttentionStack, policy_for  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--frames", type=int, default=200)
ap.add_argument("--layers", type=int, default=24)
ap.add_argument("--tau", type=float, default=0.0)
ap.add_argument("--rho", type=float, default=0.75)
ap.add_argument("--specials", type=int, default=5)
ap.add_argument("--dense", action="store_true", help="also time the dense (cuDNN SDPA) stack")
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--fused", action="store_true",
                help="also time mode='fused' (own QKV GEMM with pooled epilogue, no pool/pack passes)")
a = ap.parse_args()

torch.cuda.set_device(0)
lay = TokenLayout(a.frames, 1369, a.specials)
stack = GlobalAttentionStack(layers=a.layers)
pol = policy_for(lay, a.tau, a.rho)
g = torch.Generator(device="cuda").manual_seed(0)
x = torch.randn((lay.total_tokens, stack.dim), generator=g, device="cuda").to(torch.bfloat16)


def timed(mode):
    with torch.no_grad():
        stack(x, lay, pol, mode)  # warm-up
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.reps):
            y = stack(x, lay, pol, mode)
        e1.record()
        torch.cuda.synchronize()
    return e0.elapsed_time(e1) / a.reps, y


ms_sparse, ys = timed("sparse")
res = {"config": "24-layer VGGT global-attention stack (random init), block-sparse attention",
       "frames": a.frames, "tokens": lay.total_tokens, "layers": a.layers, "tau": a.tau,
       "rho": a.rho, "ms_per_forward": ms_sparse, "ms_per_layer": ms_sparse / a.layers,
       "frames_per_s": a.frames / (ms_sparse * 1e-3), "finite": bool(torch.isfinite(ys).all())}
if a.fused:
    ms_fused, yf = timed("fused")
    res.update({"fused_ms_per_forward": ms_fused, "fused_ms_per_layer": ms_fused / a.layers,
                "fused_frames_per_s": a.frames / (ms_fused * 1e-3),
                "fused_vs_sparse_rel_diff": float((yf.float() - ys.float()).norm() / ys.float().norm())})
if a.dense:
    ms_dense, yd = timed("dense")
    res.update({"dense_ms_per_forward": ms_dense, "dense_ms_per_layer": ms_dense / a.layers,
                "speedup_vs_dense": ms_dense / ms_sparse})
print(json.dumps(res), flush=True)
