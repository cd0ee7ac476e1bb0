"""Dense kernels of the post-pass, on the GPU in float64.

Same contracts as the reference's ``linalg.py`` (/root/reference/pkg/src/
streampca/linalg.py): the seeded Gaussian draw (``gaussian_matrix``
:46-56) is the reference's own numpy Philox generator, run on the host so
Omega is bit-identical; QR with nonnegative diag(R) (:71-98), the
triangular solve with its singularity guard (:121-136), the thin SVD
(:110-118) and the component sign convention (:156-169) run on the device
(cuSOLVER/cuBLAS through torch; tall-skinny shapes only).
"""

from __future__ import annotations

from dataclasses import dataclass

import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

from .device import default_device, to_device64, torch_mod
from .errors import (
    ConfigError,
    DataError,
    DimensionError,
    RankDeficiencyError,
    SingularMatrixError,
)

# linalg.py:26 and :31-35
RANK_TOL = 1e-12
STREAM_SKETCH = 0
STREAM_COSKETCH = 1
STREAM_FACTOR_U = 2
STREAM_FACTOR_V = 3
STREAM_REPAIR = 4


def gaussian_matrix(rows: int, cols: int, seed: int, stream: int = STREAM_SKETCH) -> np.ndarray:
    """i.i.d. N(0,1) (rows x cols) float64 from Philox keyed by (seed, stream)
    — numpy's generator, exactly as the reference draws it, so Omega (and
    therefore every result) is comparable bit for bit."""
    if rows < 1 or cols < 1:
        raise DimensionError(f"gaussian_matrix needs positive dims, got {rows}x{cols}")
    if seed < 0 or stream < 0:
        raise ConfigError("seed and stream must be nonnegative")
    key = np.array([seed, stream], dtype=np.uint64)
    n = rows * cols
    threads = min(_DRAW_THREADS, n // _DRAW_MIN_PER_THREAD)
    if threads >= 2:
        out = _parallel_normals(key, n, threads)
        if out is not None:
            return out.reshape(rows, cols)
    return np.random.Generator(np.random.Philox(key=key)).standard_normal((rows, cols))


def gaussian_matrix_device(rows: int, cols: int, seed: int, stream: int = STREAM_SKETCH, device=None):
    """gaussian_matrix drawn on the GPU (spca_gaussian_device, csrc/omega_rng.cuh):
    the same values bit for bit — numpy's Philox4x64-10 stream and float64
    ziggurat, tables recovered from numpy (ziggurat.py) — as a CUDA float64
    tensor, with no host draw and no upload (config 5's 50 M values: ~70 ms
    on 16 host cores plus a 400 MB copy). When the device cannot vouch for
    every value (a sampler test within 1e-12 of its threshold) it draws on
    the host and uploads instead."""
    import ctypes
    from . import _lib
    from .ziggurat import tables
    if rows < 1 or cols < 1:
        raise DimensionError(f"gaussian_matrix needs positive dims, got {rows}x{cols}")
    if seed < 0 or stream < 0:
        raise ConfigError("seed and stream must be nonnegative")
    torch = torch_mod()
    dev = default_device(device)
    out = torch.empty((rows, cols), dtype=torch.float64, device=dev)
    w, k, f, r_tail, inv_r = tables()
    lib = _lib.load()
    vp = ctypes.c_void_p
    with torch.cuda.device(dev):
        st = torch.cuda.current_stream(dev).cuda_stream or 1
        rc = lib.spca_gaussian_device(vp(out.data_ptr()), rows * cols, seed, stream, w.ctypes.data_as(vp),
                                      k.ctypes.data_as(vp), f.ctypes.data_as(vp), r_tail, inv_r, vp(st))
    if rc == _lib.ERR_STATE:
        return to_device64(gaussian_matrix(rows, cols, seed, stream), dev)
    _lib.check(rc)
    return out


_DRAW_THREADS = max(1, min(16, os.cpu_count() or 1))
_DRAW_MIN_PER_THREAD = 1 << 17
_OVERLAP = 64
# raw 64-bit draws per value of numpy's ziggurat standard_normal (measured:
# 1.0220616 over 2e7 values) and the lower-bound margin around the estimate
_DRAWS_PER_VALUE = 1.02206
_MARGIN = 1 << 16
_DRAW_POOL = None  # created on first use, reused by every draw (thread start-up is not free)


def _draw_pool():
    global _DRAW_POOL
    if _DRAW_POOL is None:
        _DRAW_POOL = ThreadPoolExecutor(_DRAW_THREADS, thread_name_prefix="spca-omega")
    return _DRAW_POOL


def _parallel_normals(key, n: int, threads: int):
    """The first n values of Generator(Philox(key)).standard_normal, bit for
    bit, drawn by `threads` threads (numpy releases the GIL while it fills).

    The ziggurat consumes a variable number of raw 64-bit draws per value
    (1 on its fast path, 1.022 on average), so segment t cannot be started at
    its exact counter position. Its thread starts at a lower bound instead —
    _MARGIN (65 536) raw draws before the expected position 1.022 s_t of value
    s_t, rounded down to a Philox block of four draws; the spread of the true
    position is ~sqrt(s_t)/5 draws (~1 500 at 5e7), so the bound holds with a
    wide margin — and over-generates by 2 _MARGIN (every thread draws about
    n / threads values). Every attempt of the ziggurat restarts on a fresh
    draw, so the thread's sequence of attempts merges with the true one within
    a few values; segment t - 1 also produces the first _OVERLAP values of
    segment t, and matching that run of doubles locates value s_t in thread
    t's output exactly. A segment whose run is not found (its attempts never
    merged inside the window) returns None and the caller draws serially."""
    seg = -(-n // threads)
    starts = [t * seg for t in range(threads)]
    counts = [min(seg, n - s0) for s0 in starts]
    lens, outs, raw0 = [], [None] * threads, []
    for t, s0 in enumerate(starts):
        # value s0 sits near raw draw _DRAWS_PER_VALUE * s0 (std ~ sqrt(s0) / 5):
        # start _MARGIN draws before that estimate and run 2 _MARGIN past the
        # segment, so every thread draws about the same number of values
        r0 = 0 if t == 0 else max(0, int(_DRAWS_PER_VALUE * s0) - _MARGIN) // 4 * 4
        raw0.append(r0)
        lens.append(counts[t] + _OVERLAP + (0 if t == 0 else 2 * _MARGIN + 64))

    def draw(t):
        bg = np.random.Philox(key=key)
        if t:
            bg.advance(raw0[t] // 4)
        outs[t] = np.random.Generator(bg).standard_normal(lens[t])

    pool = _draw_pool() if threads <= _DRAW_THREADS else ThreadPoolExecutor(threads)
    list(pool.map(draw, range(threads)))
    offs = [0]
    for t in range(1, threads):
        prev = outs[t - 1]
        run = prev[offs[t - 1] + counts[t - 1]: offs[t - 1] + counts[t - 1] + _OVERLAP]
        window = outs[t][: lens[t] - counts[t] - _OVERLAP + 1]
        hit = None
        for j in np.flatnonzero(window == run[0]):
            if np.array_equal(outs[t][j: j + _OVERLAP], run):
                hit = int(j)
                break
        if hit is None:
            return None
        offs.append(hit)
    out = np.empty(n)

    def place(t):
        out[starts[t]: starts[t] + counts[t]] = outs[t][offs[t]: offs[t] + counts[t]]

    list(pool.map(place, range(threads)))
    if pool is not _DRAW_POOL:
        pool.shutdown()
    return out


@dataclass(frozen=True)
class QrPair:
    q: object
    r: object


def qr_unpivoted(y, rank_check: bool = True, device=None) -> QrPair:
    """Thin Householder QR on the GPU with diag(R) >= 0 (linalg.py:71-98)."""
    torch = torch_mod()
    dev = default_device(device if device is not None else (y.device if hasattr(y, "device") and getattr(y, "is_cuda", False) else None))
    y = to_device64(y, dev)
    if y.dim() != 2:
        raise DimensionError("qr_unpivoted expects a 2-d array")
    m, b = y.shape
    if b < 1 or m < b:
        raise DimensionError(f"qr_unpivoted needs m >= b >= 1, got {m}x{b}")
    qr = _cholesky_qr2(y) if m >= 64 * b else None
    if qr is not None:
        q, r = qr
    else:
        q, r = torch.linalg.qr(y, mode="reduced")
        sign = torch.where(torch.diagonal(r) < 0, -1.0, 1.0).to(torch.float64)
        q = q * sign
        r = r * sign[:, None]
    if rank_check:
        tol = RANK_TOL * float(torch.linalg.norm(y, dim=0).max())
        small = torch.abs(torch.diagonal(r)) < tol
        if bool(small.any()):
            j = int(torch.nonzero(small)[0, 0])
            raise RankDeficiencyError(
                f"column {j} of the QR input is numerically dependent "
                f"(|r_jj| = {abs(float(r[j, j])):.3e} < tol = {tol:.3e})", column=j)
    return QrPair(q=q, r=r)


def _cholesky_qr2_flagged(y):
    """CholeskyQR2 without the host decision: (q, r, ok) with ok a device
    bool (the acceptance test of _cholesky_qr2). For pipelines that check
    many factorizations with one synchronization at the end."""
    torch = torch_mod()
    b = y.shape[1]
    eye = torch.eye(b, dtype=y.dtype, device=y.device)
    r1, info1 = torch.linalg.cholesky_ex(y.T @ y, upper=True)
    q1 = torch.linalg.solve_triangular(r1, y, upper=True, left=False)
    w2 = q1.T @ q1
    defect = torch.abs(w2 - eye).max()
    r2, info2 = torch.linalg.cholesky_ex(w2, upper=True)
    q = torch.linalg.solve_triangular(r2, q1, upper=True, left=False)
    r = r2 @ r1
    ok = (info1 == 0) & (info2 == 0) & (defect < 1e-5) & torch.isfinite(r).all() & torch.isfinite(defect)
    return q, r, ok


def _cholesky_qr2(y):
    """Thin QR of a tall, well-conditioned y by CholeskyQR2: R1 = chol(y^T y),
    Q1 = y R1^-1, then once more on Q1; R = R2 R1. Two GEMM-shaped sweeps
    over y instead of cuSOLVER's column-by-column Householder panels (the
    tall QRs of blocked_qb: 1 000 000 x 10 blocks at config 3). The result is
    the thin QR with positive diag(R) — the one the reference's sign flip
    (linalg.py:85-87) selects — to rounding. Returns None (the caller falls
    back to Householder) when y is not well conditioned: Cholesky breakdown,
    or a first-pass orthogonality defect above 1e-5 (~ u * cond(y)^2, so
    cond(y) up to ~2e5 passes, where the two factorizations agree to ~1e-11;
    every block the deficiency test could flag, |r_jj| below 1e-12 of the
    largest G column, goes to Householder)."""
    q, r, ok = _cholesky_qr2_flagged(y)
    if not bool(ok):  # one host synchronization per QR
        return None
    return q, r


@dataclass(frozen=True)
class SvdTriple:
    u: object
    s: object
    v: object


def dense_svd(b, device=None) -> SvdTriple:
    """Thin SVD of the l x n sketch factor B on the GPU (linalg.py:110-118).

    Wide B is reduced first: B^T = Q_b R_b (tall QR: CholeskyQR2 when B is
    well conditioned, else cuSOLVER Householder), then the l x l SVD
    R_b^T = U S W^T gives B = U S (Q_b W)^T — backward stable, as LAPACK's
    dgesdd does for wide inputs."""
    torch = torch_mod()
    dev = default_device(device if device is not None else (b.device if getattr(b, "is_cuda", False) else None))
    b = to_device64(b, dev)
    if b.dim() != 2 or b.shape[0] < 1 or b.shape[1] < 1:
        raise DimensionError("dense_svd expects a nonempty 2-d array")
    p, n = b.shape
    gram_ok = False
    if n >= 4 * p:
        # any non-finite entry of B leaves a non-finite entry in B B^T, so a
        # finite Gram matrix spares the n-long check (an overflowing Gram of a
        # finite B only skips the Gram route)
        w = b @ b.T
        gram_ok = bool(torch.isfinite(w).all())
        if gram_ok:
            tri = _gram_svd(b, w)
            if tri is not None:
                return tri
    if not gram_ok and not bool(torch.isfinite(b).all()):
        raise DataError("dense_svd input contains non-finite entries")
    if n > 2 * p:
        qr = _cholesky_qr2(b.T) if n >= 64 * p else None        # well conditioned: two GEMM sweeps
        qb, rb = qr if qr is not None else torch.linalg.qr(b.T, mode="reduced")  # n x p, p x p
        u, s, wt = torch.linalg.svd(rb.T, full_matrices=False)
        v = qb @ wt.T
    else:
        u, s, vt = torch.linalg.svd(b, full_matrices=False)
        v = vt.T
    return SvdTriple(u=u, s=s, v=v)


def _gram_svd(b, w=None):
    """Thin SVD of a wide, well-conditioned B (p x n, n >> p) from its Gram
    matrix: B B^T = U S^2 U^T (p x p symmetric eigenproblem), V = B^T U S^-1 —
    two GEMM sweeps over B and a p x p eigensolver instead of a tall QR of
    B^T plus a p x p SVD. The Gram squares the condition number, so it is
    taken only when every singular value is within a factor 100 of the
    largest (relative errors then ~ eps * 1e4 ~ 1e-12 on S); otherwise None
    and the QR route runs (the sketches of all five BASELINE configs have
    cond(B) < 3). V^T V = S^-1 U^T (B B^T) U S^-1 is checked on the p x p
    side (U^T W U against S^2, U^T U against I: the eigensolver's accuracy;
    forming V adds ~eps cond(B) on top), not with a third n-long GEMM.
    Orientation of each pair (u_j, v_j) is left to sign_align, as the
    reference's dgesdd output is."""
    torch = torch_mod()
    if w is None:
        w = b @ b.T
    evals, evecs = torch.linalg.eigh(w)  # ascending
    lmax = evals[-1]
    ok = (lmax > 0) & (evals[0] > 1e-4 * lmax) & torch.isfinite(evals).all()
    s = torch.sqrt(torch.clamp(evals.flip(0), min=0.0))
    u = evecs.flip(1)
    v = (b.T @ u) / s
    eye = torch.eye(b.shape[0], dtype=b.dtype, device=b.device)
    vtv = (u.T @ w @ u) / (s[:, None] * s[None, :])
    defect = torch.maximum(torch.abs(vtv - eye).max(), torch.abs(u.T @ u - eye).max())
    ok = ok & (defect < 1e-9)
    if not bool(ok):  # one host synchronization
        return None
    return SvdTriple(u=u, s=s, v=v)


def solve_rt(r, m):
    """Solve r^T x = m (r upper triangular) with the reference's singularity
    guard: any |r_jj| < 1e-300 or < 1e-15 max|r_jj| (linalg.py:121-136)."""
    torch = torch_mod()
    if r.dim() != 2 or r.shape[0] != r.shape[1]:
        raise DimensionError("solve_rt expects a square triangular matrix")
    if m.shape[0] != r.shape[0]:
        raise DimensionError(f"solve_rt shape mismatch: r is {tuple(r.shape)}, rhs has {m.shape[0]} rows")
    diag = torch.abs(torch.diagonal(r))
    scale = float(diag.max()) if r.shape[0] else 0.0
    if scale == 0.0 or bool((diag < 1e-300).any()) or bool((diag < 1e-15 * scale).any()):
        j = int(torch.argmin(diag))
        raise SingularMatrixError(f"triangular factor has near-zero diagonal at {j}")
    return torch.linalg.solve_triangular(r.T, m, upper=False)


def sign_align(u, v):
    """Flip each (u_j, v_j) so the largest-|.| entry of v_j is positive;
    first index wins ties (linalg.py:156-169)."""
    torch = torch_mod()
    idx = torch.argmax(torch.abs(v), dim=0)
    pick = v.gather(0, idx[None, :])[0]
    sign = torch.where(pick < 0, -1.0, 1.0).to(v.dtype)
    return u * sign, v * sign
