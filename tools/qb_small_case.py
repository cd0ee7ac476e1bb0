import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_1704_07669_b200 import qb as QB
rng = np.random.default_rng(0)
m, n, l, b = (int(x) for x in sys.argv[1:5]) if len(sys.argv) > 4 else (640, 100, 20, 10)
g = torch.from_numpy(rng.standard_normal((m, l))).cuda()
h = torch.from_numpy(rng.standard_normal((n, l))).cuda()
om = torch.from_numpy(rng.standard_normal((n, l))).cuda()
f = QB._blocked_qb_fused(g, h, om, b, torch.device("cuda"))
torch.cuda.synchronize()
lib = QB._blocked_qb_optimistic(g, h, om, b, torch.device("cuda"))
print("ok", f is not None, float((f.q - lib.q).abs().max()) if f is not None else None)
