"""numpy restatement of the reference single-pass PCA path (CPU oracle).

TEST INFRASTRUCTURE ONLY — see ``oracle/__init__.py``. Every function names
the reference lines it restates. Everything computes in float64, as the
reference does (``linalg.py:1-8``).

Third-party arithmetic the reference relies on (no lock file; the image pins
numpy 2.3.5 / OpenBLAS 0.3.30 and scipy 1.18.1):
  * numpy ``Philox`` bit generator + ``Generator.standard_normal`` (ziggurat)
    for Omega, used directly here exactly as ``linalg.py:39-56`` does;
  * LAPACK dgeqrf/dorgqr (``np.linalg.qr``), dgesdd (``np.linalg.svd``) and
    dtrtrs (``scipy.linalg.solve_triangular``) for the post-pass.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Iterable, Iterator, Optional

import numpy as np
import scipy.linalg

__all__ = [
    "RANK_TOL", "STREAM_SKETCH", "STREAM_FACTOR_U", "STREAM_FACTOR_V", "STREAM_REPAIR",
    "OracleError", "OracleDataError", "OracleFormatError", "OracleEmptyError",
    "OracleDeficiencyError", "OracleSingularError",
    "sketch_width", "gaussian", "row_blocks", "oracle_sketch", "oracle_center", "oracle_normalize_rows",
    "qr_pos", "solve_upper_t", "thin_svd", "align_signs", "oracle_qb",
    "oracle_single_pass", "oracle_basic_rand_svd", "oracle_legacy_single_pass",
    "oracle_lstsq", "STREAM_COSKETCH", "OracleSketch", "OracleQb", "OracleSvd",
    "synth_lowrank_plus_noise", "reference_synth_matrix", "subspace_angle",
]

# linalg.py:26 — relative rank threshold on |r_jj|
RANK_TOL = 1e-12
# linalg.py:31-35 — Philox substream ids
STREAM_SKETCH = 0
STREAM_COSKETCH = 1
STREAM_FACTOR_U = 2
STREAM_FACTOR_V = 3
STREAM_REPAIR = 4


class OracleError(Exception):
    pass


class OracleDataError(OracleError):
    def __init__(self, msg, row=None):
        super().__init__(msg)
        self.row = row


class OracleFormatError(OracleError):
    pass


class OracleEmptyError(OracleError):
    pass


class OracleDeficiencyError(OracleError):
    def __init__(self, msg, column=None, block=None):
        super().__init__(msg)
        self.column = column
        self.block = block


class OracleSingularError(OracleError):
    pass


def sketch_width(k: int, oversample: int, block_size: int) -> int:
    """algorithms.py:80-83: l = b * ceil((k + p) / b)."""
    return block_size * math.ceil((k + oversample) / block_size)


def gaussian(rows: int, cols: int, seed: int, stream: int = STREAM_SKETCH) -> np.ndarray:
    """linalg.py:39-56: Philox keyed by (seed, stream), standard normals,
    float64, C order. This *is* numpy's generator; nothing is re-derived."""
    if rows < 1 or cols < 1:
        raise OracleFormatError("gaussian needs positive dims")
    if seed < 0 or stream < 0:
        raise OracleFormatError("seed/stream must be nonnegative")
    bitgen = np.random.Philox(key=np.array([seed, stream], dtype=np.uint64))
    return np.random.Generator(bitgen).standard_normal((rows, cols))


def row_blocks(a: np.ndarray, block_rows: int) -> Iterator[tuple[int, np.ndarray]]:
    """streams.py:55-80 (ArrayRowStream.blocks): consecutive row slabs of
    an in-memory matrix widened to float64."""
    a = np.asarray(a, dtype=np.float64)
    if block_rows < 1:
        raise OracleFormatError("block_rows must be >= 1")
    for r0 in range(0, a.shape[0], block_rows):
        yield r0, a[r0:r0 + block_rows]


@dataclass(frozen=True)
class OracleSketch:
    g: np.ndarray
    h: np.ndarray
    col_sums: np.ndarray
    rows_seen: int


def oracle_sketch(
    blocks: Iterable[tuple[int, np.ndarray]],
    omega: np.ndarray,
    fixed_order: bool = False,
    compensated: bool = False,
) -> OracleSketch:
    """sketch.py:52-116 + _check_block sketch.py:40-49.

    Per block: shape check, first non-finite row -> error with absolute row;
    blocked path G_b = A_b Omega, H += A_b^T G_b, col_sums += 1^T A_b;
    fixed_order path does one gemv + rank-1 update per row; compensated
    switches col_sums to Kahan summation (per block sum, or per row in the
    fixed-order path).
    """
    om = np.asarray(omega, dtype=np.float64)
    if om.ndim != 2:
        raise OracleFormatError("omega must be 2-d")
    n, l = om.shape
    h = np.zeros((n, l))
    cs = np.zeros(n)
    carry = np.zeros(n) if compensated else None
    pieces = []
    seen = 0

    def kahan_add(total, carry, x):
        y = x - carry
        t = total + y
        return t, (t - total) - y

    for r0, vals in blocks:
        vals = np.asarray(vals, dtype=np.float64)
        if vals.ndim != 2 or vals.shape[1] != n:
            raise OracleFormatError(f"block at row {r0}: shape {vals.shape}, want (*, {n})")
        finite_rows = np.isfinite(vals).all(axis=1)
        if not finite_rows.all():
            bad = r0 + int(np.argmin(finite_rows))
            raise OracleDataError(f"non-finite value in row {bad}", row=bad)
        if fixed_order:
            gb = np.empty((vals.shape[0], l))
            for i, row in enumerate(vals):
                grow = row @ om
                gb[i] = grow
                h += row[:, None] * grow[None, :]
                if carry is None:
                    cs += row
                else:
                    cs, carry = kahan_add(cs, carry, row)
        else:
            gb = vals @ om
            h += vals.T @ gb
            bsum = vals.sum(axis=0)
            if carry is None:
                cs += bsum
            else:
                cs, carry = kahan_add(cs, carry, bsum)
        pieces.append(gb)
        seen += vals.shape[0]
    g = np.vstack(pieces) if pieces else np.zeros((0, l))
    return OracleSketch(g=g, h=h, col_sums=cs, rows_seen=seen)


def oracle_normalize_rows(vals: np.ndarray) -> np.ndarray:
    """sketch.py:142-153: subtract each row's mean, divide by the centered
    row's Euclidean norm; a zero norm divides by 1 (constant rows -> 0)."""
    x = np.asarray(vals, dtype=np.float64)
    c = x - x.mean(axis=1, keepdims=True)
    nrm = np.sqrt((c * c).sum(axis=1, keepdims=True))
    return c / np.where(nrm == 0.0, 1.0, nrm)


def oracle_center(st: OracleSketch, omega: np.ndarray) -> OracleSketch:
    """sketch.py:119-139: mu = col_sums/m; G -= 1 (mu^T Omega);
    H -= mu (1^T G); col_sums become zero."""
    if st.rows_seen == 0:
        raise OracleEmptyError("cannot center a sketch of zero rows")
    om = np.asarray(omega, dtype=np.float64)
    mu = st.col_sums / st.rows_seen
    g = st.g - np.outer(np.ones(st.rows_seen), mu @ om)
    h = st.h - np.outer(mu, st.g.sum(axis=0))
    return OracleSketch(g=g, h=h, col_sums=np.zeros_like(st.col_sums), rows_seen=st.rows_seen)


def qr_pos(y: np.ndarray, rank_check: bool = True) -> tuple[np.ndarray, np.ndarray]:
    """linalg.py:71-98: thin Householder QR with diag(R) made nonnegative by
    flipping the matching Q columns; optional rank check at
    RANK_TOL * max column norm."""
    y = np.asarray(y, dtype=np.float64)
    m, b = y.shape
    if b < 1 or m < b:
        raise OracleFormatError("qr needs m >= b >= 1")
    q, r = np.linalg.qr(y)
    flip = np.where(np.diag(r) < 0.0, -1.0, 1.0)
    q = q * flip
    r = r * flip[:, None]
    if rank_check:
        tol = RANK_TOL * float(np.max(np.linalg.norm(y, axis=0)))
        small = np.abs(np.diag(r)) < tol
        if small.any():
            raise OracleDeficiencyError("dependent column", column=int(np.argmax(small)))
    return q, r


def solve_upper_t(r: np.ndarray, rhs: np.ndarray) -> np.ndarray:
    """linalg.py:121-136: solve R^T X = rhs (R upper triangular), refusing
    diagonals below 1e-300 or 1e-15 * max|diag|."""
    d = np.abs(np.diag(r))
    top = float(d.max()) if d.size else 0.0
    if top == 0.0 or np.any(d < 1e-300) or np.any(d < 1e-15 * top):
        raise OracleSingularError(f"near-zero diagonal at {int(np.argmin(d))}")
    return scipy.linalg.solve_triangular(r, rhs, trans="T", lower=False)


@dataclass(frozen=True)
class OracleSvd:
    u: np.ndarray
    s: np.ndarray
    v: np.ndarray


def thin_svd(b: np.ndarray) -> OracleSvd:
    """linalg.py:110-118: np.linalg.svd(full_matrices=False), v = vt^T."""
    b = np.asarray(b, dtype=np.float64)
    if not np.all(np.isfinite(b)):
        raise OracleDataError("non-finite entries in the SVD input")
    u, s, vt = np.linalg.svd(b, full_matrices=False)
    return OracleSvd(u=u, s=s, v=vt.T)


def align_signs(u: np.ndarray, v: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """linalg.py:156-169: make the largest-|.| entry of every v_j positive,
    flipping u_j with it (first index wins ties, as argmax does)."""
    u = np.array(u, dtype=np.float64, copy=True)
    v = np.array(v, dtype=np.float64, copy=True)
    idx = np.argmax(np.abs(v), axis=0)
    neg = v[idx, np.arange(v.shape[1])] < 0.0
    v[:, neg] *= -1.0
    u[:, neg] *= -1.0
    return u, v


@dataclass(frozen=True)
class OracleQb:
    q: np.ndarray
    b: np.ndarray
    repaired_columns: tuple


def oracle_qb(
    g: np.ndarray,
    h: np.ndarray,
    omega: np.ndarray,
    b: int,
    reorth: bool = True,
    on_deficiency: str = "error",
    repair_seed: int = 0,
) -> OracleQb:
    """qb.py:59-171. For block i with columns c:
        Y = G[:, c] - Q (B Omega_c);  Q_i, R_i = qr_pos(Y)
        deficient if |r_jj| < RANK_TOL * max_j ||G[:, j]||   (qb.py:51-56,100)
        else (reorth) Q_i, Rt = qr_pos(Q_i - Q(Q^T Q_i)); R_i = Rt R_i
             B_i = R_i^{-T} (H[:, c]^T - (Y^T Q) B - (Omega_c^T B^T) B)
        repair (qb.py:138-171): keep the leading good columns, fill the rest
        with Philox(repair_seed, STREAM_REPAIR+i) normals orthogonalised twice
        against the basis, zero B rows.
    Q and B are preallocated instead of regrown (same arithmetic)."""
    g = np.asarray(g, dtype=np.float64)
    h = np.asarray(h, dtype=np.float64)
    om = np.asarray(omega, dtype=np.float64)
    m, l = g.shape
    n = h.shape[0]
    if h.shape[1] != l or om.shape != (n, l):
        raise OracleFormatError("inconsistent sketch shapes")
    if b < 1 or l % b:
        raise OracleFormatError("sketch width not a multiple of block size")
    if on_deficiency not in ("error", "repair"):
        raise OracleFormatError("unknown deficiency policy")
    q_all = np.zeros((m, l))
    b_all = np.zeros((l, n))
    repaired = []
    scale = float(np.max(np.linalg.norm(g, axis=0))) if g.size else 0.0

    def orth_step(y, qi, ri, q, bm, hc, oc):
        if reorth:
            q2, r2 = qr_pos(qi - q @ (q.T @ qi), rank_check=False)
            qi, ri = q2, r2 @ ri
        rhs = hc.T - (y.T @ q) @ bm - (oc.T @ bm.T) @ bm
        return qi, solve_upper_t(ri, rhs)

    for i in range(l // b):
        c0, c1 = i * b, (i + 1) * b
        q, bm = q_all[:, :c0], b_all[:c0]
        oc = om[:, c0:c1]
        y = g[:, c0:c1] - q @ (bm @ oc)
        q_y, r_y = qr_pos(y, rank_check=False)
        small = np.abs(np.diag(r_y)) < RANK_TOL * scale
        if not small.any():
            qi, bi = orth_step(y, q_y, r_y, q, bm, h[:, c0:c1], oc)
        elif on_deficiency == "error":
            j = int(np.argmax(small))
            raise OracleDeficiencyError("rank-deficient residual block",
                                        column=c0 + j, block=i)
        else:
            good = int(np.argmax(small))
            if good:
                # the reference's repair path always re-orthogonalises
                qg, rg = qr_pos(y[:, :good], rank_check=False)
                q2, r2 = qr_pos(qg - q @ (q.T @ qg), rank_check=False)
                qg, rg = q2, r2 @ rg
                rhs = (h[:, c0:c0 + good].T - (y[:, :good].T @ q) @ bm
                       - (oc[:, :good].T @ bm.T) @ bm)
                bg = solve_upper_t(rg, rhs)
            else:
                qg, bg = np.zeros((m, 0)), np.zeros((0, n))
            fill = b - good
            z = gaussian(m, fill, repair_seed, STREAM_REPAIR + i)
            basis = np.hstack([q, qg])
            for _ in range(2):
                z = z - basis @ (basis.T @ z)
            qf, _ = qr_pos(z, rank_check=False)
            qi = np.hstack([qg, qf])
            bi = np.vstack([bg, np.zeros((fill, n))])
            repaired.extend(range(c0 + good, c1))
        q_all[:, c0:c1] = qi
        b_all[c0:c1] = bi
    return OracleQb(q=q_all, b=b_all, repaired_columns=tuple(repaired))


def oracle_single_pass(
    a,
    k: int,
    oversample: int = 10,
    block_size: int = 10,
    seed: int = 0,
    center: bool = False,
    block_rows: Optional[int] = None,
    fixed_order: bool = False,
    on_deficiency: str = "repair",
    compensated: bool = False,
    omega: Optional[np.ndarray] = None,
):
    """algorithms.py:165-204 + _finish algorithms.py:144-162 over an
    in-memory matrix. Returns (u, s, v, mean, sketch, omega).

    ``omega`` may be passed to run the identical algorithm with the test
    matrix a low-precision device path actually used (e.g. fp32-rounded)."""
    a = np.asarray(a, dtype=np.float64)
    m, n = a.shape
    l = sketch_width(k, oversample, block_size)
    if m == 0:
        raise OracleEmptyError("no rows")
    if k > min(m, n) or l > min(m, n):
        raise OracleFormatError("k or l exceeds min(m, n)")
    om = gaussian(n, l, seed, STREAM_SKETCH) if omega is None else np.asarray(omega, np.float64)
    st = oracle_sketch(row_blocks(a, block_rows or l), om, fixed_order, compensated)
    mean = st.col_sums / st.rows_seen if center else None
    if center:
        st = oracle_center(st, om)
    qb = oracle_qb(st.g, st.h, om, block_size, on_deficiency=on_deficiency, repair_seed=seed)
    sv = thin_svd(qb.b)
    u, v = align_signs(qb.q @ sv.u[:, :k], sv.v[:, :k])
    return u, sv.s[:k].copy(), v, mean, st, om


def oracle_basic_rand_svd(a, k: int, oversample: int = 10, block_size: int = 10, seed: int = 0,
                          center: bool = False, block_rows: Optional[int] = None,
                          omega: Optional[np.ndarray] = None):
    """algorithms.py:207-263, the two-pass yardstick: pass 1 G = A Omega and
    col_sums per block (:230-237), optional centering of G (:241-244),
    Q = orth(G) without rank check (:245), pass 2 B += Q_i^T A_i (:247-250),
    centering of B (:251-252), SVD of B, U = Q U~ and the sign convention
    (:254-257). Returns (u, s, v, mean, q, b, omega)."""
    a = np.asarray(a, dtype=np.float64)
    m, n = a.shape
    l = sketch_width(k, oversample, block_size)
    if m == 0:
        raise OracleEmptyError("no rows")
    if k > min(m, n) or l > min(m, n):
        raise OracleFormatError("k or l exceeds min(m, n)")
    om = gaussian(n, l, seed, STREAM_SKETCH) if omega is None else np.asarray(omega, np.float64)
    br = block_rows or l
    parts, col_sums = [], np.zeros(n)
    for _, vals in row_blocks(a, br):
        parts.append(vals @ om)
        col_sums += vals.sum(axis=0)
    g = np.vstack(parts)
    mean = None
    if center:
        mean = col_sums / m
        g = g - np.outer(np.ones(m), mean @ om)
    q, _ = qr_pos(g, rank_check=False)
    bm = np.zeros((l, n))
    for r0, vals in row_blocks(a, br):
        bm += q[r0:r0 + vals.shape[0]].T @ vals
    if center:
        bm -= np.outer(q.sum(axis=0), mean)
    sv = thin_svd(bm)
    u, v = align_signs(q @ sv.u[:, :k], sv.v[:, :k])
    return u, sv.s[:k].copy(), v, mean, q, bm, om


def oracle_lstsq(lhs: np.ndarray, rhs: np.ndarray) -> np.ndarray:
    """np.linalg.lstsq(lhs, rhs, rcond=None) as algorithms.py:364 calls it:
    LAPACK dgelsd, the minimum-norm solution with singular values below
    eps * max(M, N) * s_max treated as zero."""
    return np.linalg.lstsq(lhs, rhs, rcond=None)[0]


def oracle_legacy_single_pass(a, k: int, oversample: int = 10, block_size: int = 10, seed: int = 0,
                              center: bool = False, block_rows: Optional[int] = None,
                              omega: Optional[np.ndarray] = None,
                              omega_t: Optional[np.ndarray] = None):
    """algorithms.py:312-392, the two-sketch one-pass baseline: per block
    Y_i = A_i Omega, Yt += A_i^T Omega_t[rows] and col_sums (:340-348);
    centering of Y and Yt (:353-357); Q = orth(Y), Qt = orth(Yt) (:359-360);
    core = lstsq(Omega_t^T Q, Yt^T Qt) (:361-363); cond of the system
    (:366); SVD of the core, U = Q U~, V = Qt V~, sign convention
    (:374-378). Omega_t is Philox(seed, STREAM_COSKETCH) m x l.
    Returns (u, s, v, mean, cond, y, yt)."""
    a = np.asarray(a, dtype=np.float64)
    m, n = a.shape
    l = sketch_width(k, oversample, block_size)
    if m == 0:
        raise OracleEmptyError("no rows")
    if k > min(m, n) or l > min(m, n):
        raise OracleFormatError("k or l exceeds min(m, n)")
    om = gaussian(n, l, seed, STREAM_SKETCH) if omega is None else np.asarray(omega, np.float64)
    ot = gaussian(m, l, seed, STREAM_COSKETCH) if omega_t is None else np.asarray(omega_t, np.float64)
    parts, yt, col_sums = [], np.zeros((n, l)), np.zeros(n)
    for r0, vals in row_blocks(a, block_rows or l):
        parts.append(vals @ om)
        yt += vals.T @ ot[r0:r0 + vals.shape[0]]
        col_sums += vals.sum(axis=0)
    y = np.vstack(parts)
    mean = None
    if center:
        mean = col_sums / m
        y = y - np.outer(np.ones(m), mean @ om)
        yt = yt - np.outer(mean, ot.sum(axis=0))
    q, _ = qr_pos(y, rank_check=False)
    qt, _ = qr_pos(yt, rank_check=False)
    lhs = ot.T @ q
    core = oracle_lstsq(lhs, yt.T @ qt)
    cond = float(np.linalg.cond(lhs))
    sv = thin_svd(core)
    u, v = align_signs(q @ sv.u[:, :k], qt @ sv.v[:, :k])
    return u, sv.s[:k].copy(), v, mean, cond, y, yt


def reference_synth_matrix(rows: int, cols: int, sigma: np.ndarray, seed: int) -> np.ndarray:
    """synthetic.py:141-164 + row_block :128-135 for a spectrum given as an
    explicit vector: U = Q(gauss(rows, r; seed, 2)), V = Q(gauss(cols, r;
    seed, 3)) with the rank-checked positive-diagonal QR, w = diag(sigma)V^T,
    one gemv per row. Run under a 1-thread BLAS for the reference's bytes."""
    sigma = np.asarray(sigma, dtype=np.float64)
    r = sigma.shape[0]
    u, _ = qr_pos(gaussian(rows, r, seed, STREAM_FACTOR_U))
    v, _ = qr_pos(gaussian(cols, r, seed, STREAM_FACTOR_V))
    w = sigma[:, None] * v.T
    out = np.empty((rows, cols))
    for i in range(rows):
        out[i] = u[i] @ w
    return out


def synth_lowrank_plus_noise(m: int, n: int, rank: int, spectrum: str, noise: float,
                             seed: int, dtype=np.float32) -> np.ndarray:
    """BASELINE.json configs 2/3/5 construction on the host (small sizes):
    A = X diag(s) Y^T + noise * N(0,1) with X ~ N(0,1)/sqrt(m) (m x r) and
    Y ~ N(0,1)/sqrt(n) (n x r), rounded to ``dtype``. Not in the reference
    (SURVEY.md §8(d)); used for parity cases of the fp32 path."""
    rng = np.random.Generator(np.random.Philox(key=np.array([seed, 7], dtype=np.uint64)))
    i = np.arange(1, rank + 1, dtype=np.float64)
    s = {"inv": 1.0 / i, "exp30": np.exp(-i / 30.0), "pow15": i ** -1.5,
         "invsqrt": 1.0 / np.sqrt(i)}[spectrum]
    x = rng.standard_normal((m, rank)) / math.sqrt(m)
    y = rng.standard_normal((n, rank)) / math.sqrt(n)
    a = (x * s) @ y.T + noise * rng.standard_normal((m, n))
    return a.astype(dtype)


def subspace_angle(x: np.ndarray, y: np.ndarray) -> float:
    """Largest principal angle (radians) between range(x) and range(y)."""
    ang = scipy.linalg.subspace_angles(np.asarray(x, np.float64), np.asarray(y, np.float64))
    return float(np.max(ang)) if ang.size else 0.0
