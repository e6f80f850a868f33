"""A/B of the fused scoring kernel (bsa_scoresel.cu) against the three-kernel
path: masks, counts and probabilities must be bit-identical; prints
predict_mask times for both.

    python scripts/scoresel_ab.py            # spawns both arms, compares
    python scripts/scoresel_ab.py --arm X    # one arm (BSA_SCORESEL from env)
"""
import argparse
import os
import subprocess
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

CASES = [
    # (name, frames, patches, specials, heads, d, dtype, tau, rho, seed)
    ("n200_bf16_s75", 200, 1369, 5, 16, 64, "bf16", 0.0, 0.75, 0),
    ("n200_bf16_cdf", 200, 1369, 5, 4, 64, "bf16", 0.4, 0.8, 1),
    ("n200_f32_cdf9", 200, 1369, 5, 2, 64, "f32", 0.9, 0.5, 2),
    ("n100_f32", 100, 1369, 5, 4, 64, "f32", 0.0, 0.5, 3),
    ("n300_bf16", 300, 1369, 4, 4, 64, "bf16", 0.0, 0.75, 4),
    ("n8_f32", 8, 1369, 5, 16, 64, "f32", 0.0, 0.75, 5),
    ("n8_cdf", 8, 1369, 5, 16, 64, "f32", 0.5, 0.3, 6),
    ("n30_d32", 30, 1369, 5, 3, 32, "f32", 0.3, 0.6, 7),
    ("n3_small", 3, 100, 2, 2, 16, "f32", 0.0, 0.5, 8),
    ("n1000_bf16", 1000, 1369, 5, 2, 64, "bf16", 0.0, 0.75, 9),
    ("n50_rho0", 50, 1369, 5, 2, 64, "bf16", 0.2, 0.0, 10),
    ("n50_rho1", 50, 1369, 5, 2, 64, "bf16", 0.0, 1.0, 11),
    ("n50_tau1", 50, 1369, 5, 2, 64, "f32", 1.0, 0.9, 12),
]


def run_arm(out):
    import paper_2509_07120_b200 as bsa
    res = {}
    for name, F, P, S, H, d, dt, tau, rho, seed in CASES:
        lay = bsa.TokenLayout(F, P, S)
        g = bsa.BlockGeometry(lay.patch_tokens, 128, 64)
        pol = bsa.MaskPolicy(tau, rho, g)
        gen = torch.Generator(device="cuda")
        gen.manual_seed(seed)
        dtype = torch.bfloat16 if dt == "bf16" else torch.float32
        q, k = (torch.randn((H, lay.total_tokens, d), generator=gen, device="cuda").to(dtype)
                for _ in range(2))
        mask, probs = bsa.predict_mask(q, k, pol, layout=lay, return_probs=True)
        bits = mask.device_bits().cpu().numpy()
        cnt = mask.device_counts().cpu().numpy()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 10 if F <= 300 else 3
        e0.record()
        for _ in range(reps):
            bsa.predict_mask(q, k, pol, layout=lay)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        res[name + "/bits"] = bits
        res[name + "/counts"] = cnt
        res[name + "/probs"] = probs.cpu().numpy() if F <= 300 else probs[:, :64].cpu().numpy()
        res[name + "/ms"] = np.array([ms])
        print(f"  {name}: predict_mask {ms:.3f} ms", flush=True)
        del q, k, probs
    np.savez(out, **res)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--arm")
    a = ap.parse_args()
    if a.arm:
        run_arm(a.arm)
        return
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    files = {}
    for arm, env in (("legacy", "0"), ("fused", "1")):
        f = os.path.join("/tmp", f"scoresel_{arm}.npz")
        print(f"arm {arm} (BSA_SCORESEL={env})", flush=True)
        subprocess.run([sys.executable, __file__, "--arm", f], check=True,
                       env=dict(os.environ, BSA_SCORESEL=env))
        files[arm] = np.load(f)
    bad = 0
    for name, *_ in CASES:
        A, B = files["legacy"], files["fused"]
        same = all(np.array_equal(A[name + s], B[name + s]) for s in ("/bits", "/counts"))
        psame = np.array_equal(A[name + "/probs"].view(np.uint32), B[name + "/probs"].view(np.uint32))
        bad += (not same) or (not psame)
        print(f"{name:16s} mask {'OK ' if same else 'DIFF'} probs {'OK ' if psame else 'DIFF'}  "
              f"legacy {A[name + '/ms'][0]:.3f} ms  fused {B[name + '/ms'][0]:.3f} ms")
    print("ALL BIT-IDENTICAL" if not bad else f"{bad} CASES DIFFER")
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
