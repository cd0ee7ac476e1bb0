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
buf = np.zeros(256 * STRIDE + 4 * 2048, dtype=np.uint64)
_lib.check(lib.spca_debug_trace(sk.h, 0, buf.ctypes.data, buf.size), sk.h)
t = buf[:256 * STRIDE].reshape(256, STRIDE).astype(np.int64)
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

# per unit kind (replicates fused_decode for the single launch of this run)
def sched(m, n, R0, U=int(os.environ.get("SPCA_TC_UNIT_KB", "32"))):
    kp = 2 if l <= 64 else 1  # K blocks per MMA-warp iteration (TcCfg::KP): kseg / hseg are multiples
    nkb = -(-n // 32); S = min(-(-nkb // U), 37); kseg = -(-(-(-nkb // S)) // kp) * kp; S = -(-nkb // kseg)
    nt = R0 // 128; T = nt // 2; nx = -(-n // 128); X = -(-nx // 2)
    rkb = R0 // 32; RS = -(-rkb // max(U, 48)); hseg = -(-(-(-rkb // RS)) // kp) * kp; RS = -(-rkb // hseg)
    C = -(-m // R0); rows_last = m - (C - 1) * R0; ntl = -(-rows_last // 128); Tl = -(-ntl // 2)
    return dict(C=C, T=T, Tl=Tl, S=S, X=X, RS=RS)


def kind_of(s, u):
    TS, XR = s["T"] * s["S"], s["X"] * s["RS"]
    g0 = (s["Tl"] if s["C"] == 1 else s["T"]) * s["S"]
    if u < g0:
        return 0, 0
    u -= g0
    F = TS + XR
    nmid = max(0, s["C"] - 2)
    if u < nmid * F:
        st = 1 + u // F
        r = u - (st - 1) * F
        return (0, st) if r < TS else (1, st - 1)
    u -= nmid * F
    TlS = s["Tl"] * s["S"]
    if s["C"] >= 2 and u < TlS + XR:
        return (0, s["C"] - 1) if u < TlS else (1, s["C"] - 2)
    return 1, s["C"] - 1


R0 = sk.chunk_rows()
sc = sched(rows, n, R0)
ncl = len(t) // 2


def host_order_kinds(s, lag=float(os.environ.get("SPCA_TC_LAGF", "1.0" if l <= 64 else "2.0"))):
    # the host-built unit order of tc_unit_order (tc_host.cuh): G units of chunk
    # c at c*P + r, H units at c*P + TS + lag*P + r + 0.25, stable sort
    TS, XR = s["T"] * s["S"], s["X"] * s["RS"]
    TlS = s["Tl"] * s["S"]
    P = TS + XR
    keys = []
    for c in range(s["C"]):
        g = TlS if c == s["C"] - 1 else TS
        keys += [(c * P + r, 0) for r in range(g)]
        keys += [(c * P + TS + lag * P + r + 0.25, 1) for r in range(XR)]
    keys.sort(key=lambda kv: kv[0])
    return [k for _, k in keys]


order = host_order_kinds(sc)
kinds = np.full(u.shape[:2], -1)
for cta in range(len(t)):
    for i in range(UNITS):
        uu = (cta // 2) + i * ncl
        if uu < len(order):
            kinds[cta, i] = order[uu]
mmv = (u[:, :, 5] > 0) & (u[:, :, 6] > 0)
for k, nm in ((0, "G"), (1, "H")):
    stat(f"{nm} units: MMA issue span (leader)", np.where(mmv & (kinds == k), u[:, :, 6] - u[:, :, 5], np.nan).ravel())
for k, nm in ((0, "G"), (1, "H")):
    sel = valid & (kinds == k)
    stat(f"{nm} units: epilogue duration", np.where(sel, u[:, :, 4] - u[:, :, 3], np.nan).ravel())
    stat(f"{nm} units: staging waits for epilogue", np.where(sel, u[:, :, 3] - u[:, :, 2], np.nan).ravel())
    stat(f"{nm} units: converter main loop", np.where(sel, u[:, :, 1] - u[:, :, 0], np.nan).ravel())
    stat(f"{nm} units: B producer ready - conv start", np.where(sel & (u[:, :, 7] > 0), u[:, :, 7] - u[:, :, 0], np.nan).ravel())

# leader of pair 0: per K block, time spent in each MMA-warp wait
mt = buf[256 * STRIDE:256 * STRIDE + 4 * 2048].reshape(2048, 4).astype(np.int64)
mt = mt[mt[:, 0] > 0]
if len(mt) > 2:
    nxt = np.roll(mt[:, 0], -1)
    d = np.diff(mt, axis=1) / 1e3
    issue = (nxt - mt[:, 3])[:-1] / 1e3
    per = (nxt - mt[:, 0])[:-1] / 1e3
    ok = (per > 0) & (per < 9)  # drop unit boundaries
    med = lambda x: np.median(x[:-1][ok]) if x.ndim == 1 and len(x) > len(ok) else np.median(x[ok])
    print(f"MMA warp (x1000 cycles), {ok.sum()} K blocks: per block med {np.median(per[ok]):.3f}; waits med "
          f"acc_empty {np.median(d[:-1, 0][ok]):.3f} t_full {np.median(d[:-1, 1][ok]):.3f} "
          f"b_full {np.median(d[:-1, 2][ok]):.3f}; issue+commit {np.median(issue[ok]):.3f} us; "
          f"sum of means: waits {d[:-1][ok].sum(axis=0).round(0)} issue {issue[ok].sum():.0f} us")

# converter thread 0 of CTA 0 (group 0): per K block of its own
off = 256 * STRIDE + 4 * 2048
cb = np.zeros(6 * 1024, dtype=np.uint64)
full = np.zeros(off + 6 * 1024, dtype=np.uint64)
_lib.check(lib.spca_debug_trace(sk.h, 0, full.ctypes.data, full.size), sk.h)
ct = full[off:].reshape(1024, 6).astype(np.int64)
ct = ct[ct[:, 0] > 0]
if len(ct) > 2:
    d = np.diff(ct, axis=1)
    per = np.diff(ct[:, 0])
    ok = (per > 0) & (per < 20000)
    names = ["a_full wait", "load+split+kb_empty wait", "tmem st", "wait::st", "arrive"]
    print("converter (cycles, median): per own block %d; " % np.median(per[ok]) +
          ", ".join(f"{nm} {np.median(d[:-1, i][ok]):.0f}" for i, nm in enumerate(names)) +
          "; loop rest %d" % np.median((np.roll(ct[:, 0], -1) - ct[:, 5])[:-1][ok]))

# MMA completion times (pair 0 leader), against the MMA warp's issue times
off2 = 256 * STRIDE + 4 * 2048 + 6 * 1024
full2 = np.zeros(off2 + 2048, dtype=np.uint64)
_lib.check(lib.spca_debug_trace(sk.h, 0, full2.ctypes.data, full2.size), sk.h)
done = full2[off2:].astype(np.int64)
iss = full2[256 * STRIDE:256 * STRIDE + 4 * 2048].reshape(2048, 4).astype(np.int64)[:, 3]
n_ = min((done > 0).sum(), (iss > 0).sum())
if n_ > 10:
    done, iss = done[:n_], iss[:n_]
    gap = np.diff(done)
    ok = (gap > 0) & (gap < 20000)
    lat = done - iss
    print(f"MMA completions: per block med {np.median(gap[ok]):.0f} cycles (p10 {np.percentile(gap[ok], 10):.0f}); "
          f"issue->completion med {np.median(lat):.0f} p90 {np.percentile(lat, 90):.0f} cycles")

# block-level chain for even blocks (converter group 0, thread 0 of CTA 0):
# converter arrive(k) -> MMA issue(k) -> MMA complete(k) -> converter arrive(k + NS) (stage reuse)
conv = full[off:off + 6 * 1024].reshape(1024, 6).astype(np.int64)  # own blocks 0,2,4,... (index gk>>1)
arr = conv[:, 5]
issue_t = full2[256 * STRIDE:256 * STRIDE + 4 * 2048].reshape(2048, 4).astype(np.int64)[:, 3]
comp = full2[off2:off2 + 2048].astype(np.int64)
rows = []
NS = 4
for j in range(8, 1000):
    k = 2 * j
    if k + NS >= 2048 or arr[j] == 0 or issue_t[k] == 0 or comp[k] == 0:
        continue
    jr = (k + NS) // 2
    if arr[jr] == 0:
        continue
    rows.append((issue_t[k] - arr[j], comp[k] - issue_t[k], arr[jr] - comp[k]))
if rows:
    r = np.array(rows)
    ok = np.all((r > -5000) & (r < 20000), axis=1)
    print("stage chain (cycles, median): conv arrive->MMA issue %d, issue->complete %d, complete->conv arrive(k+NS) %d"
          % tuple(np.median(r[ok], axis=0)))

# MMA waits by block position inside its unit (pair 0): where do the stalls sit?
def unit_nk(s, n_, R0_, u_):
    kind, c = kind_of(s, u_)
    nkb_ = -(-n_ // 32); U = 32
    S_ = -(-nkb_ // U); kseg_ = -(-nkb_ // S_)
    if kind == 0:
        TS = s["T"] * s["S"]
        # recover segment index b from the unit's position (approximation: full chunks)
        return kind, None
    return kind, None

mtall = full2[256 * STRIDE:256 * STRIDE + 4 * 2048].reshape(2048, 4).astype(np.int64)
valid_m = mtall[:, 0] > 0
if valid_m.sum() > 100:
    # unit boundaries: the SPCA_TRACE(ui, 5) stamp is at kb == 0 of each unit; use the gap
    # structure instead: acc_empty waits happen at kb % 4 == 0; report by (gkb mod 32)
    waits = np.diff(mtall[:, :4], axis=1)
    pos = np.arange(2048) % 32
    for p_ in (0, 1, 2, 3, 4, 8, 16, 31):
        sel = valid_m & (pos == p_)
        if sel.sum():
            w = waits[sel]
            print(f"  block pos {p_:2d}: mean acc_empty {w[:, 0].mean():6.0f} kb_full {w[:, 1].mean():6.0f} "
                  f"b_full {w[:, 2].mean():6.0f} cycles")
