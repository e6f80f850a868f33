"""Time the fused QKV projection (qkv.qkv_projection: tcgen05 GEMM + pooled
epilogue) against cuBLAS F.linear (+ the pooling the scorer then does), and
one stack layer in mode "sparse" vs "fused", at the bench shape (N frames,
16 heads x d64).  CUDA events, warm, median of reps.  Prints one JSON line."""
import argparse
import json
import os
import sys

import torch
import torch.nn.functional as F

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_07120_b200 as bsa  # noqa: E402
from paper_2509_07120_b200.stack import GlobalAttentionStack, policy_for  # noqa: E402


def timeit(fn, reps):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    return ts[len(ts) // 2]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=200)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--layer", action="store_true")
    a = ap.parse_args()
    lay = bsa.TokenLayout(a.frames, 1369, 5)
    H, C = 16, 1024
    T = lay.total_tokens
    g = torch.Generator(device="cpu").manual_seed(0)
    x = torch.randn((T, C), generator=g).to("cuda", torch.bfloat16)
    w = (torch.randn((3 * C, C), generator=g) / 32).to("cuda", torch.bfloat16)
    b = torch.zeros(3 * C, device="cuda", dtype=torch.bfloat16)
    geo = bsa.geometry_for(lay)
    Ts = lay.special_tokens
    flops = 2.0 * T * C * 3 * C
    res = {"frames": a.frames, "tokens": T, "gemm_tflop": flops / 1e12}

    res["cublas_linear_ms"] = timeit(lambda: F.linear(x, w, b), a.reps)

    def cublas_and_pool():
        y = F.linear(x, w, b).view(T, 3, H, 64).permute(1, 2, 0, 3)
        bsa.block_pool(y[0][:, Ts:], 128, validate=False)
        bsa.block_pool(y[1][:, Ts:], 64, validate=False)
    res["cublas_plus_pool_ms"] = timeit(cublas_and_pool, a.reps)
    res["fused_ms"] = timeit(lambda: bsa.qkv_projection(x, w, b, H, lay, geo), a.reps)
    res["fused_nopool_ms"] = timeit(lambda: bsa.qkv_projection(x, w, b, H, lay, geo, pooled=False),
                                    a.reps)
    res["fused_tflops"] = flops / res["fused_ms"] / 1e9
    # output projection + residual: cuBLAS linear on the transposed
    # attention output + add, vs proj_residual on the head-major output
    o = torch.randn((H, T, 64), generator=g).to("cuda", torch.bfloat16)
    wp = (torch.randn((C, C), generator=g) / 32).to("cuda", torch.bfloat16)
    bp = torch.zeros(C, device="cuda", dtype=torch.bfloat16)
    res["proj_cublas_ms"] = timeit(
        lambda: x + F.linear(o.permute(1, 0, 2).reshape(T, C), wp, bp), a.reps)
    res["proj_fused_ms"] = timeit(lambda: bsa.proj_residual(o, wp, bp, x), a.reps)
    res["cublas_tflops"] = flops / res["cublas_linear_ms"] / 1e9
    if a.layer:
        st = GlobalAttentionStack(layers=1, heads=H, seed=1)
        pol = policy_for(lay, 0.0, 0.75)
        blk = st.blocks[0]
        perm, _ = bsa.partition_permutation(lay)
        xp = x.index_select(0, torch.from_numpy(perm).cuda())
        res["layer_sparse_ms"] = timeit(lambda: st.attention(x, blk, lay, pol, "sparse"), 3)
        res["layer_fused_ms"] = timeit(lambda: st.attention_fused(xp, blk, lay, pol), 3)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
