"""Where does the bench step's time go beyond predict_mask + the attention
kernel?  Replays bench.py's step at N=200 with CUDA events between the
calls and host timestamps around them (host blocking shows up as host time
~ device time)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_07120_b200 as bsa  # noqa: E402

TIMING = len(sys.argv) > 1 and sys.argv[1] == "timing"
torch.cuda.set_device(0)
lay = bsa.TokenLayout(200, 1369, 5)
H, d = 16, 64
g = torch.Generator(device="cuda").manual_seed(0)
q, k, v = (torch.randn((H, lay.total_tokens, d), generator=g, device="cuda").to(torch.bfloat16)
           for _ in range(3))
pol = bsa.MaskPolicy(0.0, 0.75, bsa.geometry_for(lay))


def step(ev):
    h = [time.perf_counter()]
    ev[0].record()
    mask = bsa.predict_mask(q, k, pol, layout=lay)
    ev[1].record()
    h.append(time.perf_counter())
    job = bsa.SparseAttentionJob(bsa.AttentionInputs(q, k, v), lay, mask)
    ev[2].record()
    h.append(time.perf_counter())
    out = bsa.sparse_attention(job, timing=TIMING)
    ev[3].record()
    h.append(time.perf_counter())
    return out, h


for _ in range(3):
    step([torch.cuda.Event(enable_timing=True) for _ in range(4)])
torch.cuda.synchronize()
rows = []
evs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(5)]
t0 = time.perf_counter()
hs = []
for i in range(5):
    _, h = step(evs[i])
    if TIMING:
        h.append(bsa.sparse.last_kernel_ms())
    hs.append(h)
torch.cuda.synchronize()
t1 = time.perf_counter()
for i in range(5):
    e = evs[i]
    dev = [e[0].elapsed_time(e[1]), e[1].elapsed_time(e[2]), e[2].elapsed_time(e[3])]
    gap = evs[i][3].elapsed_time(evs[i + 1][0]) if i < 4 else 0.0
    h = hs[i]
    print(f"step {i}: device predict {dev[0]:.3f} inputs {dev[1]:.3f} attention {dev[2]:.3f} "
          f"gap-to-next {gap:.3f} | host predict {1e3*(h[1]-h[0]):.3f} inputs {1e3*(h[2]-h[1]):.3f} "
          f"attention {1e3*(h[3]-h[2]):.3f} ms" + (f" | kernel {h[4]:.3f}" if TIMING else ""))
print(f"wall per step {1e3*(t1-t0)/5:.3f} ms; events first->last {evs[0][0].elapsed_time(evs[4][3])/5:.3f} ms")
