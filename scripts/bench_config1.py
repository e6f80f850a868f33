"""BASELINE.json config 1: one layer at N=8 frames, fp32, the reference's
default-ish policy (tau=0.4, rho=0.8) -- the fp32 path: bit-exact fp32
scoring and fp32-accurate attention (<= 1e-4 max-abs) on the tensor cores
(split-bf16 X3 kernel, the default) or on the CUDA cores (path="simt").
Also times the same layer through the bf16 tensor-core path and reports the
fp32 paths' max-abs difference from a float64 reference. Prints JSON.
FRAMES=<n> in the environment changes N."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_07120_b200 as bsa  # noqa: E402

lay = bsa.TokenLayout(int(os.environ.get("FRAMES", "8")), 1369, 5)
rng = np.random.default_rng(0)
q, k, v = (rng.standard_normal((16, lay.total_tokens, 64)).astype(np.float32) for _ in range(3))
pol = bsa.MaskPolicy(0.4, 0.8, bsa.BlockGeometry(lay.patch_tokens, 128, 64))
res = {"config": f"N={lay.frames} frames (T={lay.total_tokens}), 16 heads x d64, tau=0.4 rho=0.8"}
outs = {}
for dt, path in (("fp32", "auto"), ("fp32_simt", "simt"), ("bf16", "auto")):
    tdt = torch.float32 if dt.startswith("fp32") else torch.bfloat16
    dq, dk, dv = (torch.from_numpy(x).to("cuda", tdt) for x in (q, k, v))

    def step():
        mask = bsa.predict_mask(dq, dk, pol, layout=lay)
        job = bsa.SparseAttentionJob(bsa.AttentionInputs(dq, dk, dv), lay, mask)
        return bsa.sparse_attention(job, path=path), mask

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
    res[dt] = {"ms_per_layer": e0.elapsed_time(e1) / 10, "path": bsa.attention_path(job, path),
               "achieved_sparsity": float(mask.achieved_sparsity().mean())}
    if dt.startswith("fp32"):
        outs[dt] = (out.float().cpu().numpy() if torch.is_tensor(out) else np.asarray(out)), mask
if lay.frames <= 8:
    import oracle  # test infrastructure: the float64 checker (not timed)
    for dt, (o, mk) in outs.items():
        ref = oracle.masked_attention_f64(q, k, v, lay.frames, 1369, 5, mk.blocks, 128, 64)
        res[dt]["max_abs_vs_f64"] = float(np.abs(o - ref).max())
print(json.dumps(res))
