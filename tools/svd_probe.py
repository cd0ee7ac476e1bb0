"""Time dense_svd / finish_svd alone on a config-shaped B (l x n fp64).
    python tools/svd_probe.py [cfg] [reps]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1704_07669_b200.linalg import dense_svd
from paper_1704_07669_b200.synth import config_shape

cfg_name = sys.argv[1] if len(sys.argv) > 1 else "cfg5"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
cs = config_shape(cfg_name)
l, n = cs["l"], cs["n"]
dev = torch.device("cuda:0")
gen = torch.Generator(device=dev).manual_seed(0)
s = torch.logspace(0, -4, l, dtype=torch.float64, device=dev)
u = torch.linalg.qr(torch.randn(l, l, dtype=torch.float64, device=dev, generator=gen))[0]
v = torch.linalg.qr(torch.randn(n, l, dtype=torch.float64, device=dev, generator=gen))[0]
b = (u * s) @ v.T
for r in range(reps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = dense_svd(b)
    torch.cuda.synchronize()
    print(cfg_name, "dense_svd ms", round(1e3 * (time.perf_counter() - t0), 2), flush=True)
