"""Per-stage device times of the scoring path at the bench workload."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_07120_b200 as bsa  # noqa: E402

F = int(sys.argv[1]) if len(sys.argv) > 1 else 200
lay = bsa.TokenLayout(F, 1369, 5)
g = bsa.BlockGeometry(lay.patch_tokens, 128, 64)
gen = torch.Generator(device="cuda")
gen.manual_seed(0)
q, k = (torch.randn((16, lay.total_tokens, 64), generator=gen, device="cuda").to(torch.bfloat16)
        for _ in range(2))
pidx = torch.from_numpy(bsa.patch_token_indices(lay)).cuda()


def timed(fn, n=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        r = fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n, r


for tau, rho in [(0.0, 0.75), (0.4, 0.8), (0.9, 0.5)]:
    pol = bsa.MaskPolicy(tau, rho, g)
    qpat, kpat = q[:, pidx].contiguous(), k[:, pidx].contiguous()
    t_pool, qp = timed(lambda: bsa.block_pool(qpat, 128))
    t_poolk, kp = timed(lambda: bsa.block_pool(kpat, 64))
    t_sc, pr = timed(lambda: bsa.pooled_scores(qp, kp, 64))
    t_sel, _ = timed(lambda: bsa.select_blocks(pr, pol))
    t_all, _ = timed(lambda: bsa.predict_mask(q, k, pol, layout=lay))
    print(f"tau={tau} rho={rho}: pool q {t_pool:.3f} k {t_poolk:.3f}  scores+softmax {t_sc:.3f}  "
          f"select {t_sel:.3f}  predict_mask (fused) {t_all:.3f} ms")
