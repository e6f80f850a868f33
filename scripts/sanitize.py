"""Small-shape driver for compute-sanitizer (memcheck / racecheck / synccheck
/ initcheck) over every kernel family of libbsa.so:

  scoring     pool8/pool8a/pool, kblock + the fused scoresel kernel (tau=0
              and tau>0; BSA_SCORESEL=0: scores, pw_plan, softsel), fallback
              (forced by an unnormalised row)
  attention   pack, schedule, bsa_tc_kernel stale-max launch + exact-max
              repair launch (large logits force overflowed items), the fp32
              X3 launch + its CUDA-core repair of large-logit rows, the fp32
              SIMT kernel, the scatter epilogue (1 emulated rank)
  analysis    bsa_stats_kernel passes 1 and 2

Usage (GPU box):
  compute-sanitizer --tool racecheck python scripts/sanitize.py
Prints one line per stage; exit code 0 when every result is finite.
"""

from __future__ import annotations

import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2509_07120_b200 as bsa  # noqa: E402
from paper_2509_07120_b200 import analysis  # noqa: E402


def qkv(h, t, d, seed, scale=1.0):
    g = torch.Generator(device="cuda")
    g.manual_seed(seed)
    return [torch.randn((h, t, d), generator=g, device="cuda") * scale for _ in range(3)]


def main():
    torch.cuda.set_device(0)
    lay = bsa.TokenLayout(2, 300, 5)
    H, d = 2, 64
    q, k, v = qkv(H, lay.total_tokens, d, 0)
    g = bsa.BlockGeometry(lay.patch_tokens, 128, 64)
    ok = True
    for tau, rho in ((0.0, 0.75), (0.4, 0.8)):
        pol = bsa.MaskPolicy(tau, rho, g)
        mask = bsa.predict_mask(q, k, pol, layout=lay)
        print(f"predict_mask tau={tau}: counts {mask.device_counts().sum().item()}", flush=True)
    # unnormalised scores force the exact fallback path of select_blocks
    s = torch.rand((1, 4, 40), device="cuda") * 1e-12
    sel = bsa.select_blocks(s, bsa.MaskPolicy(0.9, 1.0, bsa.BlockGeometry(160, 40, 4)))
    print(f"select_blocks fallback: {int(sel.device_counts().sum().item())} blocks", flush=True)

    pol = bsa.MaskPolicy(0.0, 0.75, g)
    mask = bsa.predict_mask(q, k, pol, layout=lay)
    qb, kb, vb = (x.to(torch.bfloat16) for x in (q, k, v))
    out = bsa.sparse_attention(bsa.SparseAttentionJob(bsa.AttentionInputs(qb, kb, vb), lay, mask))
    ok &= bool(torch.isfinite(out.float()).all())
    print("tc attention: finite", bool(torch.isfinite(out.float()).all()), flush=True)
    # large logits: stale offset overflows, exact-max repair launch runs
    ramp = torch.linspace(0.2, 8.0, lay.total_tokens, device="cuda")[None, :, None]
    kr = (k * 6.0 * ramp).to(torch.bfloat16)
    qr = (q * 6.0).to(torch.bfloat16)
    out = bsa.sparse_attention(bsa.SparseAttentionJob(bsa.AttentionInputs(qr, kr, vb), lay, mask))
    ok &= bool(torch.isfinite(out.float()).all())
    print("tc attention (repair launch): finite", bool(torch.isfinite(out.float()).all()), flush=True)
    job32 = bsa.SparseAttentionJob(bsa.AttentionInputs(q, k, v), lay, mask)
    out32 = bsa.sparse_attention(job32)
    ok &= bool(torch.isfinite(out32).all())
    print("fp32 tc (X3) attention: finite", bool(torch.isfinite(out32).all()), flush=True)
    out32 = bsa.sparse_attention(bsa.SparseAttentionJob(
        bsa.AttentionInputs(q * 6.0, k * 6.0 * ramp, v), lay, mask))
    ok &= bool(torch.isfinite(out32).all())
    print("fp32 tc (X3) + CUDA-core repair: finite", bool(torch.isfinite(out32).all()), flush=True)
    out32 = bsa.sparse_attention(job32, path="simt")
    ok &= bool(torch.isfinite(out32).all())
    print("simt attention: finite", bool(torch.isfinite(out32).all()), flush=True)

    from paper_2509_07120_b200.shard import DeviceOps, ShardPlan, ScatterTarget
    plan = ShardPlan(lay, 1)
    tgt = ScatterTarget(plan, H, d, 0, None, "cuda")
    DeviceOps().attend_scatter(qb, kb, vb, lay, mask, 0, 1, tgt)
    torch.cuda.synchronize()
    ok &= bool(torch.isfinite(tgt.local.float()).all())
    print("scatter epilogue: finite", bool(torch.isfinite(tgt.local.float()).all()), flush=True)
    tgt.close()

    inp = bsa.AttentionInputs(qb, kb, vb)
    rs = analysis.attention_row_stats(inp, lay)
    bm = analysis.block_attention_map(inp, lay, rs)
    ok &= bool(torch.isfinite(rs).all()) and bool(torch.isfinite(bm).all())
    print("stats kernels: finite", bool(torch.isfinite(bm).all()), flush=True)
    # fused QKV projection (tcgen05 GEMM + pooled epilogue) and scoring from the pools
    C = 4 * 64
    x = torch.randn((lay.total_tokens, C), device="cuda").to(torch.bfloat16)
    w = (torch.randn((3 * C, C), device="cuda") / 16).to(torch.bfloat16)
    b = torch.randn((3 * C,), device="cuda").to(torch.bfloat16)
    q4, k4, v4, qp4, kp4 = bsa.qkv_projection(x, w, b, 4, lay)
    m4 = bsa.predict_mask_pooled(qp4, kp4, bsa.MaskPolicy(0.4, 0.8, g))
    ok &= bool(torch.isfinite(qp4).all()) and bool(torch.isfinite(v4.float()).all())
    print(f"qkv_projection + predict_mask_pooled: {int(m4.device_counts().sum().item())} blocks",
          flush=True)
    o4 = torch.randn((4, lay.total_tokens, 64), device="cuda").to(torch.bfloat16)
    wp = (torch.randn((C, C), device="cuda") / 16).to(torch.bfloat16)
    y4 = bsa.proj_residual(o4, wp, b[:C], x)
    ok &= bool(torch.isfinite(y4.float()).all())
    print("proj_residual: finite", bool(torch.isfinite(y4.float()).all()), flush=True)
    torch.cuda.synchronize()
    print("SANITIZE_DRIVER_OK" if ok else "SANITIZE_DRIVER_BAD", flush=True)
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main())
