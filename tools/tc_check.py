"""Quick tensor-core path check: tc vs simt vs fp64 oracle on a few shapes.

    python tools/tc_check.py
"""

import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import oracle as O  # noqa: E402
import paper_1704_07669_b200 as P  # noqa: E402


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def main():
    shapes = [(128, 32, 8), (256, 64, 60), (1000, 333 * 4, 30), (3000, 1000, 60), (5000, 4096, 120),
              (700, 2000, 250), (20000, 10000, 60)]
    for (m, n, l) in shapes:
        a = O.gaussian(m, n, seed=m).astype(np.float32)
        om = O.gaussian(n, l, seed=n)
        om32 = om.astype(np.float32).astype(np.float64)
        ref = O.oracle_sketch(O.row_blocks(a, 4096), om32)
        out = {}
        for prec in ("simt", "tc"):
            t0 = time.perf_counter()
            st = P.sketch_pass(P.ArrayRowStream(a), om, precision=prec)
            dt = time.perf_counter() - t0
            out[prec] = (rel(st.g, ref.g), rel(st.h, ref.h),
                         float(np.max(np.abs(st.col_sums - ref.col_sums))), dt)
        print(f"m={m} n={n} l={l}: " + "  ".join(
            f"{p}: G {e[0]:.1e} H {e[1]:.1e} cs {e[2]:.1e} ({e[3]*1e3:.0f} ms)" for p, e in out.items()),
            flush=True)


if __name__ == "__main__":
    main()
