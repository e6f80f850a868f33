"""N=200: attention with the keys forced into 1, 2 or 3 L2-sized ranges
(sparse_attention(key_ranges=n)): kernel time (CUDA events inside the
library), whole sparse_attention call (incl. the LSE combine), alternating
settings, and parity of the outputs between settings."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_07120_b200 as bsa  # noqa: E402

torch.cuda.set_device(0)
F = int(sys.argv[1]) if len(sys.argv) > 1 else 200
lay = bsa.TokenLayout(F, 1369, 5)
H, d = 16, 64
g = torch.Generator(device="cuda").manual_seed(0)
q, k, v = (torch.randn((H, lay.total_tokens, d), generator=g, device="cuda").to(torch.bfloat16)
           for _ in range(3))
pol = bsa.MaskPolicy(0.0, 0.75, bsa.geometry_for(lay))
mask = bsa.predict_mask(q, k, pol, layout=lay)
job = bsa.SparseAttentionJob(bsa.AttentionInputs(q, k, v), lay, mask)
settings = [int(x) for x in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["1", "2", "3"])]
outs = {}
for n in settings:
    outs[n] = bsa.sparse_attention(job, key_ranges=n)
torch.cuda.synchronize()
res = {n: ([], []) for n in settings}
for rep in range(4):
    for n in settings:
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        bsa.sparse_attention(job, key_ranges=n, timing=True)
        b.record()
        kern = bsa.sparse.last_kernel_ms()
        res[n][0].append(kern)
        res[n][1].append(a.elapsed_time(b))
for n in settings:
    ref = outs[settings[0]].float()
    rel = ((outs[n].float() - ref).abs().max() / ref.abs().max()).item()
    print(f"ranges {n}: kernel ms {[round(x, 2) for x in res[n][0]]} call ms "
          f"{[round(x, 2) for x in res[n][1]]} max rel diff vs {settings[0]}: {rel:.2e}", flush=True)
