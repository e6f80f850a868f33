"""Time predict_mask and sparse_attention of the N=200 layer whole vs in
head chunks (heads are independent), to see whether chunking pays."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_07120_b200 as bsa  # noqa: E402

F = int(os.environ.get("FRAMES", 200))
lay = bsa.TokenLayout(F, 1369, 5)
g = bsa.BlockGeometry(lay.patch_tokens, 128, 64)
pol = bsa.MaskPolicy(0.0, 0.75, g)
gen = torch.Generator(device="cuda")
gen.manual_seed(0)
q, k, v = (torch.randn((16, lay.total_tokens, 64), generator=gen, device="cuda").to(torch.bfloat16)
           for _ in range(3))


def timeit(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    return ts[len(ts) // 2]


for c in (16, 8, 4, 2):
    spans = [(a, a + c) for a in range(0, 16, c)]
    masks = [bsa.predict_mask(q[a:b], k[a:b], pol, layout=lay) for a, b in spans]
    t_mask = timeit(lambda: [bsa.predict_mask(q[a:b], k[a:b], pol, layout=lay) for a, b in spans])
    jobs = [bsa.SparseAttentionJob(bsa.AttentionInputs(q[a:b], k[a:b], v[a:b]), lay, m)
            for (a, b), m in zip(spans, masks)]
    t_att = timeit(lambda: [bsa.sparse_attention(j) for j in jobs])

    def both():
        for a, b in spans:
            m = bsa.predict_mask(q[a:b], k[a:b], pol, layout=lay)
            bsa.sparse_attention(bsa.SparseAttentionJob(bsa.AttentionInputs(q[a:b], k[a:b], v[a:b]), lay, m))
    t_both = timeit(both)
    print(f"chunk={c:2d}: predict_mask {t_mask:7.2f} ms  attention {t_att:7.2f} ms  layer {t_both:7.2f} ms",
          flush=True)
