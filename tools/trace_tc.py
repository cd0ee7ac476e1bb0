"""Per-CTA timeline of the tensor-core kernels for one cfg2-like chunk.
    SPCA_TC_TRACE=1 python tools/trace_tc.py [rows] [n] [l]"""
import ctypes, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1704_07669_b200 as P
from paper_1704_07669_b200 import _lib
rows = int(sys.argv[1]) if len(sys.argv) > 1 else 46080
n = int(sys.argv[2]) if len(sys.argv) > 2 else 10000
l = int(sys.argv[3]) if len(sys.argv) > 3 else 60
a = torch.randn(rows, n, device="cuda", dtype=torch.float32)
om = np.random.default_rng(0).standard_normal((n, l))
sk = P.GpuSketch(n, om, np.float32, precision="tc", rows_hint=rows)
lib = _lib.load()
lib.spca_debug_trace.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_int64]
for rep in range(3):
    sk.reset(); sk.push(a, 0); sk.finish()
names = ["start", "setup", "tma0", "tmaN", "mma0", "mmaN", "conv0", "convN", "epi0", "epiN", "end"]
for which, kname in ((0, "G"), (1, "H")):
    buf = np.zeros(4096 * 16, dtype=np.uint64)
    _lib.check(lib.spca_debug_trace(sk.h, which, buf.ctypes.data, buf.size), sk.h)
    t = buf.reshape(-1, 16)[:, :11].astype(np.int64)
    t = t[t[:, 0] > 0]
    t0 = t[:, 0].min()
    rel = (t - t0) / 1e3
    print(f"kernel {kname}: {len(t)} CTAs, span {rel[:, 10].max():.1f} us")
    for i, nm in enumerate(names):
        col = rel[:, i]
        print(f"   {nm:6s} min {col.min():7.2f}  med {np.median(col):7.2f}  max {col.max():7.2f} us")
