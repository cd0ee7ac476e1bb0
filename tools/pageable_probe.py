"""Pass rate from pageable host memory (a plain numpy array, the reference's
usual input) vs page-locked host memory, config-2 shape.
    python tools/pageable_probe.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1704_07669_b200 as P

m, n, l = 100000, 10000, 60
a = np.random.default_rng(0).standard_normal((m, n), dtype=np.float32)
pin = torch.from_numpy(a).pin_memory()
om = P.gaussian_matrix(n, l, 1)
sk = P.GpuSketch(n, om, np.float32, rows_hint=m)
for name, src in (("pageable numpy", a), ("pinned tensor", pin)):
    ts = []
    for rep in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        sk.reset()
        sk.push(src, 0, final=True)
        sk.finish(on_device=True)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    t = min(ts)
    print(f"{name}: {t * 1e3:.1f} ms per pass, {a.nbytes / t / 1e9:.1f} GB/s")
