"""GPU timeline of one bench step (torch.profiler, CUPTI): every kernel /
memset / memcpy with start offset and duration, and the idle gaps."""
import os
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_07120_b200 as bsa  # noqa: E402

F = int(sys.argv[1]) if len(sys.argv) > 1 else 200
lay = bsa.TokenLayout(F, 1369, 5)
pol = bsa.MaskPolicy(0.0, 0.75, bsa.BlockGeometry(lay.patch_tokens, 128, 64))
g = torch.Generator(device="cuda").manual_seed(0)
q, k, v = (torch.randn((16, lay.total_tokens, 64), generator=g, device="cuda").to(torch.bfloat16)
           for _ in range(3))


def step():
    mask = bsa.predict_mask(q, k, pol, layout=lay)
    return bsa.sparse_attention(bsa.SparseAttentionJob(bsa.AttentionInputs(q, k, v), lay, mask))


for _ in range(3):
    step()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    for _ in range(2):
        step()
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
ev.sort(key=lambda e: e.time_range.start)
t0 = ev[0].time_range.start
prev_end = t0
for e in ev:
    s, d = e.time_range.start, e.time_range.end - e.time_range.start
    gap = s - prev_end
    print(f"{(s - t0) / 1e3:9.3f} ms  gap {gap / 1e3:7.3f}  dur {d / 1e3:8.3f}  {e.name[:70]}")
    prev_end = max(prev_end, e.time_range.end)
print(f"total {(prev_end - t0) / 1e3:.3f} ms for 2 steps")
