"""Device time of the dense attention statistics (analysis.py) at the bench
shapes: pass 1 (row stats over all T keys) and pass 2 (block map over the
patch keys), CUDA events, and the S FLOPs / exp2 rates they reach."""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_07120_b200 as bsa  # noqa: E402
from paper_2509_07120_b200.analysis import (  # noqa: E402
    attention_row_stats, block_attention_map, quadrant_stats_from_rows)

ap = argparse.ArgumentParser()
ap.add_argument("--frames", type=int, default=200)
ap.add_argument("--heads", type=int, default=16)
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
lay = bsa.TokenLayout(a.frames, 1369, 5)
g = torch.Generator(device="cuda").manual_seed(0)
q, k, v = (torch.randn((a.heads, lay.total_tokens, 64), generator=g, device="cuda")
           .to(torch.bfloat16) for _ in range(3))
inp = bsa.AttentionInputs(q, k, v)
T, Tp = lay.total_tokens, lay.patch_tokens


def timed(fn):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(a.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        r = fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return min(ts), r


t1, rs = timed(lambda: attention_row_stats(inp, lay))
t2, bm = timed(lambda: block_attention_map(inp, lay, row_stats=rs))
st = quadrant_stats_from_rows(rs, lay)
f1 = 2 * 64 * a.heads * T * (-(-T // 128) * 128 / T) * T  # S FLOPs incl. row padding
f2 = 2 * 64 * a.heads * Tp * Tp
print(json.dumps({
    "frames": a.frames, "heads": a.heads, "tokens": T,
    "row_stats_ms": t1, "row_stats_tflops": f1 / t1 / 1e9, "row_stats_gexp_per_s": a.heads * T * T / t1 / 1e6,
    "block_map_ms": t2, "block_map_tflops": f2 / t2 / 1e9, "block_map_gexp_per_s": a.heads * Tp * Tp / t2 / 1e6,
    "map_elements_avoided": a.heads * T * T,
    "quadrant_means_head0": {k_: float(v_[0]) for k_, v_ in st.means.items()},
    "block_map_row_mass_head0_qb0": float(bm[0, 0].sum()),
}))
