"""Kernel-time breakdown of blocked_qb on a config-shaped random sketch
(torch.profiler, CUDA activity): python tools/qb_prof.py [cfg]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import ProfilerActivity, profile

import paper_1704_07669_b200 as P
from paper_1704_07669_b200.synth import config_shape

cfg_name = sys.argv[1] if len(sys.argv) > 1 else "cfg5"
cs = config_shape(cfg_name)
m, n, l = cs["m"], cs["n"], cs["l"]
dev = torch.device("cuda:0")
gen = torch.Generator(device=dev).manual_seed(0)
g = torch.randn(m, l, dtype=torch.float64, device=dev, generator=gen)
h = torch.randn(n, l, dtype=torch.float64, device=dev, generator=gen)
om = torch.randn(n, l, dtype=torch.float64, device=dev, generator=gen)
for _ in range(2):
    P.blocked_qb(g, h, om, 10)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    P.blocked_qb(g, h, om, 10)
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=18, max_name_column_width=60))
