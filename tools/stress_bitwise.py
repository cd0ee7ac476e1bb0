"""Repeat the pass many times and require bitwise-identical G, H, col_sums
(catches rare ordering races in the persistent kernel).
    python tools/stress_bitwise.py [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1704_07669_b200 as P

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 30
shapes = [(100000, 10000, 60), (40000, 4096, 120), (6000, 200000, 250), (30000, 3000, 17)]
bad = 0
for m, n, l in shapes:
    g = torch.Generator(device="cuda").manual_seed(m + n)
    a = torch.randn((m, n), generator=g, device="cuda", dtype=torch.float32)
    om = P.gaussian_matrix(n, l, seed=3)
    sk = P.GpuSketch(n, om, np.float32, precision="tc", rows_hint=m)
    ref = None
    for r in range(reps):
        sk.reset()
        sk.push(a, 0, final=True)
        gg, hh, cs, rows = sk.finish(on_device=True)
        sig = (gg.view(torch.int64).sum().item(), hh.view(torch.int64).sum().item(),
               cs.view(torch.int64).sum().item(), bool(torch.isfinite(gg).all()))
        if ref is None:
            ref = sig
        elif sig != ref:
            bad += 1
            print(f"MISMATCH {m}x{n} l={l} rep {r}: {sig} vs {ref}", flush=True)
    sk.close()
    print(f"{m}x{n} l={l}: {reps} reps, finite={ref[3]}", flush=True)
print("mismatches:", bad)
sys.exit(1 if bad else 0)
