"""Pass time of the tensor-core path when the row stride is not a multiple of
16 bytes (re-strided through the padded buffer) vs an aligned stride.
    python tools/odd_n_probe.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1704_07669_b200 as P

for n in (10000, 10001):
    a = torch.randn(100000, n, device="cuda", dtype=torch.float32)
    om = P.gaussian_matrix(n, 60, 1)
    sk = P.GpuSketch(n, om, np.float32, precision="tc", rows_hint=100000)
    for rep in range(4):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        sk.reset()
        sk.push(a, 0, final=True)
        sk.finish(on_device=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
    print(f"n={n}: {dt * 1e3:.2f} ms per pass ({a.numel() * 4 / dt / 1e9:.0f} GB/s)")
    sk.close()
    del a
