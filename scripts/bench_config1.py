"""BASELINE.json config 1: one layer at N=8 frames, fp32, the reference's
default-ish policy (tau=0.4, rho=0.8) -- the exact-arithmetic path: bit-exact
fp32 scoring and the fp32 CUDA-core attention kernel (<= 1e-4 max-abs).
Also times the same layer through the bf16 tensor-core path. Prints JSON."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_07120_b200 as bsa  # noqa: E402

lay = bsa.TokenLayout(8, 1369, 5)
rng = np.random.default_rng(0)
q, k, v = (rng.standard_normal((16, lay.total_tokens, 64)).astype(np.float32) for _ in range(3))
pol = bsa.MaskPolicy(0.4, 0.8, bsa.BlockGeometry(lay.patch_tokens, 128, 64))
res = {"config": "N=8 frames (T=10,992), 16 heads x d64, tau=0.4 rho=0.8"}
for dt in ("fp32", "bf16"):
    tdt = torch.float32 if dt == "fp32" else torch.bfloat16
    dq, dk, dv = (torch.from_numpy(x).to("cuda", tdt) for x in (q, k, v))

    def step():
        mask = bsa.predict_mask(dq, dk, pol, layout=lay)
        job = bsa.SparseAttentionJob(bsa.AttentionInputs(dq, dk, dv), lay, mask)
        return bsa.sparse_attention(job), mask

    for _ in range(3):
        out, mask = step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        out, mask = step()
    e1.record()
    torch.cuda.synchronize()
    job = bsa.SparseAttentionJob(bsa.AttentionInputs(dq, dk, dv), lay, mask)
    res[dt] = {"ms_per_layer": e0.elapsed_time(e1) / 10, "path": bsa.attention_path(job),
               "achieved_sparsity": float(mask.achieved_sparsity().mean())}
print(json.dumps(res))
