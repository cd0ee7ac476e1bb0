import time, numpy as np, torch, sys
sys.path.insert(0, '/root/repo')
import paper_1704_07669_b200 as P
from paper_1704_07669_b200 import synth, gaussian_matrix, GpuSketch
a = synth.config_matrix("cfg2", device=torch.device("cuda", 0))
m, n = a.shape
om = gaussian_matrix(n, 60, 1)
sk = GpuSketch(n, om, np.float32, precision="tc", rows_hint=m)
for _ in range(3):
    sk.reset(); sk.push(a, 0); sk.finish(on_device=True)
torch.cuda.synchronize()
T = {"reset": [], "push": [], "finish": []}
for _ in range(10):
    t0 = time.perf_counter(); sk.reset(); torch.cuda.synchronize(); t1 = time.perf_counter()
    sk.push(a, 0, final=True); torch.cuda.synchronize(); t2 = time.perf_counter()
    sk.finish(on_device=True); torch.cuda.synchronize(); t3 = time.perf_counter()
    T["reset"].append(t1 - t0); T["push"].append(t2 - t1); T["finish"].append(t3 - t2)
print({k: round(np.median(v) * 1e3, 3) for k, v in T.items()})
