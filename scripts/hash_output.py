"""sha256 of the N=200 bench layer's output (for bit-identity checks between
library variants: BSA_LIB_VARIANT=<name>), over several runs."""
import hashlib
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_07120_b200 as bsa  # noqa: E402

frames = int(sys.argv[1]) if len(sys.argv) > 1 else 200
runs = int(sys.argv[2]) if len(sys.argv) > 2 else 3
lay = bsa.TokenLayout(frames, 1369, 5)
pol = bsa.MaskPolicy(0.0, 0.75, bsa.BlockGeometry(lay.patch_tokens, 128, 64))
g = torch.Generator(device="cuda").manual_seed(0)
q, k, v = (torch.randn((16, lay.total_tokens, 64), generator=g, device="cuda").to(torch.bfloat16)
           for _ in range(3))
mask = bsa.predict_mask(q, k, pol, layout=lay)
for r in range(runs):
    out = bsa.sparse_attention(bsa.SparseAttentionJob(bsa.AttentionInputs(q, k, v), lay, mask))
    torch.cuda.synchronize()
    h = hashlib.sha256(out.view(torch.int16).cpu().numpy().tobytes()).hexdigest()[:16]
    print(os.environ.get("BSA_LIB_VARIANT", "main"), frames, r, h, flush=True)
