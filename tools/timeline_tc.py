"""Per-chunk kernel spans of the tensor-core path (G and H kernels) for one pass.
    SPCA_TC_TRACE=1 python tools/timeline_tc.py [rows] [n] [l]"""
import ctypes, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1704_07669_b200 as P
from paper_1704_07669_b200 import _lib
rows = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
n = int(sys.argv[2]) if len(sys.argv) > 2 else 10000
l = int(sys.argv[3]) if len(sys.argv) > 3 else 60
a = torch.randn(rows, n, device="cuda", dtype=torch.float32)
om = np.random.default_rng(0).standard_normal((n, l))
sk = P.GpuSketch(n, om, np.float32, precision="tc", rows_hint=rows)
lib = _lib.load()
lib.spca_debug_trace.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_int64]
sk.reset(); sk.push(a, 0); sk.finish()  # warm (chunks 0..k-1)
nch = -(-rows // sk.chunk_rows())
W = 4096 * 16 + 4096
g = np.zeros(W, dtype=np.uint64); hb = np.zeros(W, dtype=np.uint64)
_lib.check(lib.spca_debug_trace(sk.h, 0, g.ctypes.data, W), sk.h)
_lib.check(lib.spca_debug_trace(sk.h, 1, hb.ctypes.data, W), sk.h)
tg = g[4096 * 16:].reshape(-1, 4)[:nch].astype(np.float64)
th = hb[4096 * 16:].reshape(-1, 4)[:nch].astype(np.float64)
t0 = tg[0, 0]
print(f"{nch} chunks of {sk.chunk_rows()} rows; times in us from the first G start")
for c in range(nch):
    gs, ge = (tg[c, 0] - t0) / 1e3, (tg[c, 1] - t0) / 1e3
    hs, he = (th[c, 2] - t0) / 1e3, (th[c, 3] - t0) / 1e3
    print(f"chunk {c:3d}: G [{gs:8.1f} {ge:8.1f}] {ge-gs:6.1f}   H [{hs:8.1f} {he:8.1f}] {he-hs:6.1f}   G->H gap {hs-ge:6.1f}")
print("pass span", (th[nch-1, 3] - t0) / 1e3, "us")
