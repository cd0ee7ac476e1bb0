"""Time blocked_qb alone on a config-shaped sketch (random G, H, Omega of the
config's m, n, l; the factorization does not care where they came from).
    python tools/qb_probe.py [cfg] [reps]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1704_07669_b200 as P
from paper_1704_07669_b200.synth import config_shape

cfg_name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
cs = config_shape(cfg_name)
m, n, l = cs["m"], cs["n"], cs["l"]
dev = torch.device("cuda:0")
gen = torch.Generator(device=dev).manual_seed(0)
g = torch.randn(m, l, dtype=torch.float64, device=dev, generator=gen)
h = torch.randn(n, l, dtype=torch.float64, device=dev, generator=gen)
om = torch.randn(n, l, dtype=torch.float64, device=dev, generator=gen)
for r in range(reps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    f = P.blocked_qb(g, h, om, 10)
    torch.cuda.synchronize()
    print(cfg_name, "blocked_qb ms", round(1e3 * (time.perf_counter() - t0), 2), flush=True)
