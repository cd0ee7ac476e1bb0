"""Per-CTA timeline of the pass kernel (sketch_fused.cuh) for one push.
    SPCA_TC_TRACE=1 python tools/trace_fused.py [rows] [n] [l]
Prints the kernel span and, per unit, how long each role spent: converter
main loop, converters waiting for the epilogue staging, epilogue duration,
MMA issue span, and the B producer's dependency wait (H units)."""
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
for rep in range(3):
    sk.reset(); sk.push(a, 0); sk.finish()
STRIDE, UNITS = 1024, 127
buf = np.zeros(256 * STRIDE, dtype=np.uint64)
_lib.check(lib.spca_debug_trace(sk.h, 0, buf.ctypes.data, buf.size), sk.h)
t = buf.reshape(256, STRIDE).astype(np.int64)
t = t[t[:, 0] > 0]
t0 = t[:, 0].min()
end = (t[:, 1] - t0) / 1e3
print(f"{len(t)} CTAs, kernel span {end.max():.1f} us; CTA end min {end.min():.1f} med {np.median(end):.1f}")
u = t[:, 8:8 + 8 * UNITS].reshape(len(t), UNITS, 8)
valid = (u[:, :, 0] > 0) & (u[:, :, 4] > 0)


def stat(name, x):
    x = x[np.isfinite(x)] / 1e3
    if len(x):
        print(f"  {name:34s} med {np.median(x):7.2f}  p90 {np.percentile(x, 90):7.2f}  max {x.max():7.2f} us")


stat("converter main loop", np.where(valid, u[:, :, 1] - u[:, :, 0], np.nan).ravel())
stat("converter wait for staging", np.where(valid, u[:, :, 2] - u[:, :, 1], np.nan).ravel())
nxt = np.roll(u[:, :, 0], -1, axis=1)
stat("converter gap to next unit", np.where(valid & (nxt > 0), nxt - u[:, :, 2], np.nan)[:, :-1].ravel())
stat("epilogue pickup after staging", np.where(valid, u[:, :, 3] - u[:, :, 2], np.nan).ravel())
stat("epilogue duration", np.where(valid, u[:, :, 4] - u[:, :, 3], np.nan).ravel())
mm = (u[:, :, 5] > 0) & (u[:, :, 6] > 0)
stat("MMA issue span (leader)", np.where(mm, u[:, :, 6] - u[:, :, 5], np.nan).ravel())
stat("B producer dep-wait end - conv start", np.where(valid & (u[:, :, 7] > 0), u[:, :, 7] - u[:, :, 0], np.nan).ravel())
