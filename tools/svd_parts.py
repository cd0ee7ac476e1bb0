"""Where dense_svd's time goes on a config-shaped B (the Gram route):
    python tools/svd_parts.py [cfg]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1704_07669_b200.synth import config_shape

cfg_name = sys.argv[1] if len(sys.argv) > 1 else "cfg5"
cs = config_shape(cfg_name)
l, n = cs["l"], cs["n"]
dev = torch.device("cuda:0")
gen = torch.Generator(device=dev).manual_seed(0)
s = torch.logspace(0, -1, l, dtype=torch.float64, device=dev)
u = torch.linalg.qr(torch.randn(l, l, dtype=torch.float64, device=dev, generator=gen))[0]
v = torch.linalg.qr(torch.randn(n, l, dtype=torch.float64, device=dev, generator=gen))[0]
b = (u * s) @ v.T


def lap(name, fn, reps=5):
    out = None
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        out = fn()
        torch.cuda.synchronize()
        ts.append(1e3 * (time.perf_counter() - t0))
    print(f"{cfg_name} {name:28s} ms {min(ts):8.3f} (median {sorted(ts)[len(ts)//2]:.3f})", flush=True)
    return out


w = lap("gram B B^T", lambda: b @ b.T)
ev = lap("eigh (cusolver)", lambda: torch.linalg.eigh(w))
wc = w.cpu().numpy()
lap("eigh (numpy, host)", lambda: np.linalg.eigh(wc))
lap("eigh host incl. copies", lambda: torch.from_numpy(np.linalg.eigh(w.cpu().numpy())[1]).to(dev))
uu = ev[1].flip(1)
ss = torch.sqrt(ev[0].flip(0))
vv = lap("V = B^T U / s", lambda: (b.T @ uu) / ss)
lap("defect V^T V", lambda: torch.abs(vv.T @ vv - torch.eye(l, dtype=torch.float64, device=dev)).max())
lap("isfinite(B).all()", lambda: bool(torch.isfinite(b).all()))
from paper_1704_07669_b200.linalg import dense_svd
lap("dense_svd total", lambda: dense_svd(b))
