"""Stage trace of CTA 0 of the fused scoring kernel (BSA_SCORESEL_DEBUG=2):
K-stage issue -> data ready -> consumed, in clock64 cycles."""
import ctypes
import os
import sys

os.environ["BSA_SCORESEL_DEBUG"] = "2"
import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_07120_b200 as bsa  # noqa: E402
from paper_2509_07120_b200 import _native as N  # noqa: E402

lay = bsa.TokenLayout(200, 1369, 5)
g = bsa.BlockGeometry(lay.patch_tokens, 128, 64)
pol = bsa.MaskPolicy(0.0, 0.75, g)
gen = torch.Generator(device="cuda")
gen.manual_seed(0)
q, k = (torch.randn((16, lay.total_tokens, 64), generator=gen, device="cuda").to(torch.bfloat16)
        for _ in range(2))
for _ in range(2):
    bsa.predict_mask(q, k, pol, layout=lay)
torch.cuda.synchronize()
buf = np.zeros(1536, dtype=np.uint64)
L = N.lib()
assert L.bsa_debug_scoring_trace(buf.ctypes.data, buf.nbytes) == 0
iss, rdy, con = buf[:512].astype(np.int64), buf[512:1024].astype(np.int64), buf[1024:].astype(np.int64)
n = int((rdy > 0).sum())
t0 = iss[0]
print(f"{n} stages")
print("stage  issue  ready  consumed  (cycles from first issue)  issue->ready  ready->consumed")
for s in list(range(0, min(n, 12))) + list(range(n - 4, n)):
    print(f"{s:4d} {iss[s]-t0:7d} {rdy[s]-t0:7d} {con[s]-t0:7d}   {rdy[s]-iss[s]:6d} {con[s]-rdy[s]:6d}")
d = np.diff(con[:n])
print(f"median consumed period {np.median(d):.0f} clk, median issue->ready {np.median(rdy[:n]-iss[:n]):.0f}")
