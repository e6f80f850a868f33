"""Seconds-long sanity check of a library variant (BSA_LIB_VARIANT): one
small tensor-core attention call against the float64 oracle. Exit 0 = OK.
Run it under a short `timeout` before any long benchmark of a new variant."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import paper_2509_07120_b200 as bsa  # noqa: E402

lay = bsa.TokenLayout(3, 700, 5)
rng = np.random.default_rng(0)
q, k, v = (rng.standard_normal((2, lay.total_tokens, 64)).astype(np.float32) for _ in range(3))
qd, kd, vd = (torch.from_numpy(x).to("cuda", torch.bfloat16) for x in (q, k, v))
g = bsa.BlockGeometry(lay.patch_tokens, 128, 64)
mask = bsa.predict_mask(qd, kd, bsa.MaskPolicy(0.4, 0.8, g), layout=lay)
out = bsa.sparse_attention(bsa.SparseAttentionJob(bsa.AttentionInputs(qd, kd, vd), lay, mask))
ref = oracle.masked_attention_f64(*(t.float().cpu().numpy() for t in (qd, kd, vd)), 3, 700, 5,
                                  mask.blocks, 128, 64)
err = float(np.abs(out.float().cpu().numpy() - ref).max() / np.abs(ref).max())
print(f"quick_check {os.environ.get('BSA_LIB_VARIANT', 'default')}: rel err {err:.2e}")
sys.exit(0 if err <= 2e-2 else 1)
