"""Per-chunk / per-tile error of the pass kernel's G and H with many chunks.
    SPCA_TC_CHUNK_MB=1 python tools/tc_multichunk.py [m] [n] [l]"""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1704_07669_b200 as P

m = int(sys.argv[1]) if len(sys.argv) > 1 else 5000
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
l = int(sys.argv[3]) if len(sys.argv) > 3 else 60
rng = np.random.default_rng(3)
a = rng.standard_normal((m, n)).astype(np.float32)
om = rng.standard_normal((n, l))
sk = P.GpuSketch(n, om, np.float32, precision="tc", rows_hint=m)
R0 = sk.chunk_rows()
print("chunk rows", R0, "chunks", -(-m // R0))
sk.push(torch.from_numpy(a).cuda(), 0)
g, hh, cs, _ = sk.finish(on_device=False)
a64 = a.astype(np.float64)
g_ref = a64 @ om.astype(np.float32).astype(np.float64)
err = np.abs(g - g_ref).max(axis=1) / np.abs(g_ref).max()
for c in range(-(-m // R0)):
    rows = slice(c * R0, min(m, (c + 1) * R0))
    e = err[rows]
    bad_tiles = sorted(set(int(i) // 128 for i in np.nonzero(e > 1e-5)[0]))
    print(f"chunk {c:3d}: max rel {e.max():.2e}  bad tiles {bad_tiles}")
h_ref = a64.T @ g
print("H rel err", np.abs(hh - h_ref).max() / np.abs(h_ref).max(),
      "colsum rel", np.abs(cs - a64.sum(0)).max() / np.abs(a64.sum(0)).max())

# diagnose: is the error of a bad row a stale partial of chunk c - 3 (same tile row)?
nkb = -(-n // 32)
S = -(-nkb // 32)
kseg = -(-nkb // S)
S = -(-nkb // kseg)
om32 = om.astype(np.float32).astype(np.float64)
bad_rows = np.nonzero(err > 1e-5)[0][:6]
for r in bad_rows:
    diff = g[r] - g_ref[r]
    c = r // R0
    msg = []
    for s in range(S):
        k0, k1 = s * kseg * 32, min(n, (s + 1) * kseg * 32)
        own = a64[r, k0:k1] @ om32[k0:k1]
        for back in (3, 6, 1, 2):
            if r - back * R0 >= 0:
                old = a64[r - back * R0, k0:k1] @ om32[k0:k1]
                if np.abs(diff - (old - own)).max() < 1e-3 * np.abs(own).max():
                    msg.append(f"seg {s} from chunk c-{back}")
        if np.abs(diff + own).max() < 1e-3 * np.abs(own).max():
            msg.append(f"seg {s} missing")
    print(f"row {r} (chunk {c}, tile {(r % R0) // 128}): |diff| {np.abs(diff).max():.3g} -> {msg}")
