"""Debug: with kSlots >= chunks, compare every K-split partial of the pass kernel
with the fp64 reference (tile, segment): python tools/tc_partials.py"""
import ctypes, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1704_07669_b200 as P
from paper_1704_07669_b200 import _lib
m, n, l = 20000, 10000, 60
rng = np.random.default_rng(3)
a = rng.standard_normal((m, n)).astype(np.float32)
om = rng.standard_normal((n, l))
sk = P.GpuSketch(n, om, np.float32, precision="tc", rows_hint=m)
R0 = sk.chunk_rows()
sk.push(torch.from_numpy(a).cuda(), 0)
g, hh, cs, _ = sk.finish(on_device=False)
lib = _lib.load()
lib.spca_debug_gpart.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64]
C = m // R0; nt = R0 // 128; nkb = -(-n // 32); S = -(-nkb // 32); kseg = -(-nkb // S); S = -(-nkb // kseg)
slots = 3
gp = np.zeros(slots * nt * S * 128 * 64, dtype=np.float32)
_lib.check(lib.spca_debug_gpart(sk.h, gp.ctypes.data, gp.size), sk.h)
gp = gp.reshape(slots, nt, S, 128, 64)[..., :l]
a64 = a.astype(np.float64); om32 = om.astype(np.float32).astype(np.float64)
for c in range(C):
    bad = []
    for t in range(nt):
        rows = slice(c * R0 + t * 128, c * R0 + t * 128 + 128)
        for s in range(S):
            k0, k1 = s * kseg * 32, min(n, (s + 1) * kseg * 32)
            ref = a64[rows, k0:k1] @ om32[k0:k1]
            e = np.abs(gp[c % slots, t, s] - ref).max() / np.abs(ref).max()
            if e > 1e-5:
                bad.append((t, s, round(float(e), 3)))
    gerr = np.abs(g[c * R0:(c + 1) * R0] - a64[c * R0:(c + 1) * R0] @ om32).max()
    print(f"chunk {c}: bad partials {bad[:8]}{'...' if len(bad) > 8 else ''} ({len(bad)}); G max abs err {gerr:.3g}")

# classify the first few bad partials: which K blocks / periods explain the difference?
shown = 0
for c in range(C):
    for t in range(nt):
        rows = slice(c * R0 + t * 128, c * R0 + t * 128 + 128)
        for s in range(S):
            k0, k1 = s * kseg * 32, min(n, (s + 1) * kseg * 32)
            ref = a64[rows, k0:k1] @ om32[k0:k1]
            d = gp[c % slots, t, s].astype(np.float64) - ref
            if np.abs(d).max() / np.abs(ref).max() <= 1e-5 or c == 0 or shown >= 6:
                continue
            shown += 1
            nkb_s = (k1 - k0 + 31) // 32
            X = [a64[rows, k0 + 32 * j:min(k1, k0 + 32 * j + 32)] @ om32[k0 + 32 * j:min(k1, k0 + 32 * j + 32)]
                 for j in range(nkb_s)]
            found = []
            for j in range(nkb_s):
                for sign, nm in ((-1, "missing"), (1, "doubled")):
                    if np.abs(d - sign * X[j]).max() < 1e-3 * np.abs(ref).max():
                        found.append(f"kb {j} {nm}")
            for p in range(0, nkb_s, 4):
                Xp = sum(X[p:p + 4])
                for sign, nm in ((-1, "missing"), (1, "doubled")):
                    if np.abs(d - sign * Xp).max() < 1e-3 * np.abs(ref).max():
                        found.append(f"period {p // 4} {nm}")
            # rows affected
            rows_bad = np.nonzero(np.abs(d).max(axis=1) > 1e-4 * np.abs(ref).max())[0]
            cols_bad = np.nonzero(np.abs(d).max(axis=0) > 1e-4 * np.abs(ref).max())[0]
            print(f"chunk {c} tile {t} seg {s}: rows bad {len(rows_bad)} {rows_bad[:6]}, cols bad {len(cols_bad)} {cols_bad[:6]} -> {found}")
