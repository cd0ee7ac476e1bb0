"""Merged column-group launch (l > 128) vs one launch per group: the same
sketch bit for bit (the per-group work and reduction orders are identical).
    python tools/merged_check.py [m n l]   (run once plain, once with SPCA_TC_SEQ_GROUPS=1)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1704_07669_b200 as P

m, n, l = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (6000, 3000, 250)))
gen = torch.Generator(device="cuda").manual_seed(1)
a = torch.randn(m, n, device="cuda", dtype=torch.float32, generator=gen)
om = np.random.default_rng(2).standard_normal((n, l))
sk = P.GpuSketch(n, om, np.float32, precision="tc", rows_hint=m)
sk.push(a, 0, final=True)
g, h, cs, rows = sk.finish(on_device=True)
torch.cuda.synchronize()
tag = "seq" if os.environ.get("SPCA_TC_SEQ_GROUPS") else "merged"
np.savez(f"gpurun_out/merged_check_{tag}.npz", g=g.cpu().numpy(), h=h.cpu().numpy(), cs=cs.cpu().numpy())
ref_g = a.double() @ torch.from_numpy(om.astype(np.float32).astype(np.float64)).cuda()
print(tag, "rows", rows, "rel err G", float(torch.linalg.norm(g - ref_g) / torch.linalg.norm(ref_g)))
