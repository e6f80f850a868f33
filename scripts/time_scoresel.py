"""Device time of scoring from pooled inputs (kblock + scoresel + fallback:
predict_mask_pooled) at N frames, 16 heads; BSA_SCORESEL_DEBUG=1 in the
environment skips phase B (timing only)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_07120_b200 as bsa  # noqa: E402

F = int(sys.argv[1]) if len(sys.argv) > 1 else 200
lay = bsa.TokenLayout(F, 1369, 5)
geo = bsa.geometry_for(lay)
gen = torch.Generator(device="cuda").manual_seed(0)
q, k = (torch.randn((16, lay.total_tokens, 64), generator=gen, device="cuda").to(torch.bfloat16)
        for _ in range(2))
Ts = lay.special_tokens
pidx = torch.from_numpy(bsa.patch_token_indices(lay)).cuda()
qp = bsa.block_pool(q[:, pidx].contiguous(), 128)
kp = bsa.block_pool(k[:, pidx].contiguous(), 64)
pol = bsa.MaskPolicy(0.0, 0.75, geo)
ref = bsa.predict_mask(q, k, pol, layout=lay)
m = bsa.predict_mask_pooled(qp, kp, pol)
same = bool(torch.equal(m.device_bits(), ref.device_bits()))
ts = []
for _ in range(3):
    bsa.predict_mask_pooled(qp, kp, pol)
torch.cuda.synchronize()
for _ in range(10):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    bsa.predict_mask_pooled(qp, kp, pol)
    b.record()
    b.synchronize()
    ts.append(a.elapsed_time(b))
ts.sort()
print(f"{os.environ.get('BSA_LIB_VARIANT', 'default')} debug={os.environ.get('BSA_SCORESEL_DEBUG', '0')}: "
      f"scoring from pools {ts[len(ts) // 2]:.3f} ms (min {ts[0]:.3f}), mask equal: {same}", flush=True)
