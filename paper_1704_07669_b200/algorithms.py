"""Public single-pass PCA entry point, B200 edition.

Signature- and result-compatible with the reference's ``single_pass_pca``
(/root/reference/pkg/src/streampca/algorithms.py:165-204): same
``PcaConfig`` (:52-101), same ``TruncatedSvd`` (:104-119), same Omega
(Philox(seed, STREAM_SKETCH)), same error classes. The pass runs in
libspca.so and the post-pass (blocked QB, small SVD, U = Q U~, sign
convention) runs on the GPU in float64; only U, S, V (and the mean) come
back to the host.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Optional, Union

import numpy as np

from .device import default_device, host_copy, to_device64, torch_mod
from .errors import ConfigError, EmptyStreamError
from .linalg import STREAM_SKETCH, dense_svd, gaussian_matrix_device, qr_unpivoted, sign_align
from .qb import QbFactor, blocked_qb
from .sketch import SketchState, run_pass, sketch_pass
from .streams import ArrayRowStream, PassCounter, RowStream


@dataclass(frozen=True)
class PcaConfig:
    """k, oversample, block_size, power, seed, center — the reference's knobs
    with its validation (algorithms.py:52-101); l = b * ceil((k + p) / b)."""

    k: int
    oversample: int = 10
    block_size: int = 10
    power: int = 0
    seed: int = 0
    center: bool = False

    def __post_init__(self):
        if self.k < 1:
            raise ConfigError(f"target rank k must be >= 1, got {self.k}")
        if self.oversample < 0:
            raise ConfigError(f"oversample must be >= 0, got {self.oversample}")
        if self.block_size < 1:
            raise ConfigError(f"block_size must be >= 1, got {self.block_size}")
        if self.power not in (0, 1):
            raise ConfigError(f"power must be 0 or 1, got {self.power}")
        if self.seed < 0:
            raise ConfigError(f"seed must be >= 0, got {self.seed}")

    @property
    def l(self) -> int:
        return self.block_size * math.ceil((self.k + self.oversample) / self.block_size)

    @property
    def n_blocks(self) -> int:
        return self.l // self.block_size

    def validate_dims(self, n_cols: int, n_rows: Optional[int] = None) -> None:
        limit = n_cols if n_rows is None else min(n_rows, n_cols)
        if self.k > limit:
            raise ConfigError(f"target rank k={self.k} exceeds min(m, n)={limit}")
        if self.l > limit:
            raise ConfigError(
                f"sketch width l={self.l} (k + oversample rounded up to a block multiple) "
                f"exceeds min(m, n)={limit}; lower oversample or block_size")


@dataclass(frozen=True)
class TruncatedSvd:
    """A ~ u diag(s) v^T (algorithms.py:104-119); numpy float64 arrays."""

    u: np.ndarray
    s: np.ndarray
    v: np.ndarray
    mean: Optional[np.ndarray] = None
    passes: Optional[int] = None
    retained_floats: Optional[int] = None
    warnings: tuple = ()

    @property
    def k(self) -> int:
        return int(self.s.shape[0])


MatrixOrStream = Union[np.ndarray, RowStream]


def as_row_stream(data) -> RowStream:
    """Streams pass through; arrays become ArrayRowStream (float32 kept),
    CUDA tensors DeviceRowStream, host tensors PinnedRowStream."""
    if hasattr(data, "blocks") and hasattr(data, "n_cols"):
        return data
    try:
        import torch
        if isinstance(data, torch.Tensor):
            from .streams import DeviceRowStream, PinnedRowStream
            return DeviceRowStream(data) if data.is_cuda else PinnedRowStream(data)
    except ImportError:  # pragma: no cover
        pass
    return ArrayRowStream(data)


def _measured_passes(stream, fallback: int) -> int:
    return stream.passes_completed if isinstance(stream, PassCounter) else fallback


def finish_svd(factor: QbFactor, k: int):
    """_finish (algorithms.py:144-162) on the device: SVD of B, U = Q U~[:, :k],
    V = V~[:, :k], sign convention; returns CUDA tensors (u, s, v)."""
    small = dense_svd(factor.b)
    u = factor.q @ small.u[:, :k]
    v = small.v[:, :k]
    u, v = sign_align(u, v)
    return u, small.s[:k].clone(), v


def single_pass_pca(
    data: MatrixOrStream,
    cfg: PcaConfig,
    block_rows: Optional[int] = None,
    fixed_order: bool = False,
    on_deficiency: str = "repair",
    compensated: bool = False,
    *,
    precision: str = "auto",
    device=None,
    return_device: bool = False,
) -> TruncatedSvd:
    """Truncated SVD / PCA from exactly one traversal of the rows
    (algorithms.py:165-204), sketch and post-pass on the GPU."""
    stream = as_row_stream(data)
    if cfg.power != 0:
        raise ConfigError("single_pass_pca runs at power 0; use power_refine for power 1")
    if stream.n_rows == 0:
        raise EmptyStreamError("the stream has no rows")
    cfg.validate_dims(stream.n_cols, stream.n_rows)
    dev = default_device(device)
    omega = gaussian_matrix_device(stream.n_cols, cfg.l, cfg.seed, stream=STREAM_SKETCH, device=dev)
    state = sketch_pass(stream, omega, block_rows=block_rows, fixed_order=fixed_order,
                        compensated=compensated, precision=precision, device=dev,
                        keep_on_device=True, shift=cfg.center)
    if state.rows_seen == 0:
        raise EmptyStreamError("the stream yielded no rows")
    cfg.validate_dims(stream.n_cols, state.rows_seen)
    return _post_pass(state, cfg, stream, on_deficiency, return_device, passes_fallback=1)


def _post_pass(state: SketchState, cfg: PcaConfig, stream, on_deficiency, return_device,
               passes_fallback: int) -> TruncatedSvd:
    from .sketch import center_correct
    mean = None
    if cfg.center:
        mean = state.col_sums / state.rows_seen
        state = center_correct(state, state.omega)
    factor = blocked_qb(state.g, state.h, state.omega, cfg.block_size,
                        on_deficiency=on_deficiency, repair_seed=cfg.seed)
    u, s, v = finish_svd(factor, cfg.k)
    retained = state.retained_floats + int(state.omega.numel())
    if not return_device:
        u, s, v = host_copy(u), host_copy(s), host_copy(v)
        mean = host_copy(mean) if mean is not None else None
    return TruncatedSvd(u=u, s=s, v=v, mean=mean,
                        passes=_measured_passes(stream, passes_fallback),
                        retained_floats=retained)


def power_refine(
    data: MatrixOrStream,
    cfg: PcaConfig,
    block_rows: Optional[int] = None,
    fixed_order: bool = False,
    on_deficiency: str = "repair",
    *,
    precision: str = "auto",
    device=None,
    return_device: bool = False,
) -> TruncatedSvd:
    """Power-sharpened variant (algorithms.py:266-309): pass 1 sketches with
    Omega and keeps H; Omega2 = orth(H) (on the GPU) drives pass 2 through
    the same kernels."""
    from .errors import CapabilityError
    from .sketch import center_correct
    stream = as_row_stream(data)
    if cfg.power != 1:
        raise ConfigError("power_refine requires power = 1 in the config")
    if not stream.resettable:
        raise CapabilityError("power_refine needs a resettable stream (two passes)")
    if stream.n_rows == 0:
        raise EmptyStreamError("the stream has no rows")
    cfg.validate_dims(stream.n_cols, stream.n_rows)
    dev = default_device(device)
    omega = gaussian_matrix_device(stream.n_cols, cfg.l, cfg.seed, stream=STREAM_SKETCH, device=dev)
    first = sketch_pass(stream, omega, block_rows=block_rows, precision=precision,
                        device=dev, keep_on_device=True, shift=cfg.center)
    if first.rows_seen == 0:
        raise EmptyStreamError("the stream yielded no rows")
    cfg.validate_dims(stream.n_cols, first.rows_seen)
    mean = first.col_sums / first.rows_seen if cfg.center else None
    if cfg.center:
        first = center_correct(first, first.omega)
    omega2 = qr_unpivoted(first.h, rank_check=False, device=dev).q
    second = sketch_pass(stream, omega2.cpu().numpy(), block_rows=block_rows, precision=precision,
                         device=dev, keep_on_device=True, shift=cfg.center)
    if cfg.center:
        second = center_correct(second, second.omega)
    factor = blocked_qb(second.g, second.h, second.omega, cfg.block_size,
                        on_deficiency=on_deficiency, repair_seed=cfg.seed)
    u, s, v = finish_svd(factor, cfg.k)
    retained = second.retained_floats + int(second.omega.numel())
    if not return_device:
        u, s, v = host_copy(u), host_copy(s), host_copy(v)
        mean = host_copy(mean) if mean is not None else None
    return TruncatedSvd(u=u, s=s, v=v, mean=mean, passes=_measured_passes(stream, 2),
                        retained_floats=retained)


def _finish_pair(sk):
    """Finished state of a GpuSketch as CUDA float64 tensors + rows, handle closed."""
    try:
        return sk.finish(on_device=True)
    finally:
        sk.close()


def basic_rand_svd(
    data: MatrixOrStream,
    cfg: PcaConfig,
    block_rows: Optional[int] = None,
    *,
    precision: str = "auto",
    device=None,
    return_device: bool = False,
) -> TruncatedSvd:
    """Two-pass yardstick (algorithms.py:207-263): pass 1 G = A Omega and the
    column sums; Q = orth(G) on the GPU (rank check off, :245); pass 2 the
    same kernels with Q as the co-sketch operand give H = A^T Q = B^T
    (:247-250); centering of G and B (:241-244, 251-252); SVD of B, U = Q U~,
    sign convention (:254-257)."""
    from .errors import CapabilityError
    torch = torch_mod()
    stream = as_row_stream(data)
    if not stream.resettable:
        raise CapabilityError("basic_rand_svd needs a resettable stream (two passes)")
    if stream.n_rows == 0:
        raise EmptyStreamError("the stream has no rows")
    cfg.validate_dims(stream.n_cols, stream.n_rows)
    dev = default_device(device)
    n = stream.n_cols
    omega = gaussian_matrix_device(n, cfg.l, cfg.seed, stream=STREAM_SKETCH, device=dev)
    sk = run_pass(stream, omega, block_rows=block_rows, precision=precision, device=dev, shift=cfg.center)
    try:
        g, _, col_sums, m = sk.finish(on_device=True)
        if m == 0:
            raise EmptyStreamError("the stream yielded no rows")
        cfg.validate_dims(n, m)
        om = sk.omega_used(on_device=True)
        mean = None
        if cfg.center:
            mean = col_sums / m
            g = g - (mean @ om)[None, :]
        q = qr_unpivoted(g, rank_check=False, device=dev).q
        # pass 2 on the same handle: H = A^T Q (the B^T of B += Q_i^T A_i)
        run_pass(stream, omega, block_rows=block_rows, precision=precision, device=dev, left=q, sk=sk)
        _, bt, _, m2 = sk.finish(on_device=True)
    finally:
        sk.close()
    if m2 != m:
        raise CapabilityError(f"second pass yielded {m2} rows, the first {m}")
    if cfg.center:
        bt = bt - torch.outer(mean, q.sum(dim=0))
    small = dense_svd(bt.T.contiguous())
    u, v = sign_align(q @ small.u[:, :cfg.k], small.v[:, :cfg.k])
    s = small.s[:cfg.k].clone()
    retained = int(m * cfg.l + n * cfg.l + cfg.l * n + n)  # g + omega + b + col_sums (:262)
    if not return_device:
        u, s, v = host_copy(u), host_copy(s), host_copy(v)
        mean = host_copy(mean) if mean is not None else None
    return TruncatedSvd(u=u, s=s, v=v, mean=mean, passes=_measured_passes(stream, 2),
                        retained_floats=retained)


def _lstsq_min_norm(lhs, rhs):
    """np.linalg.lstsq(lhs, rhs, rcond=None) (LAPACK dgelsd) on the device:
    the minimum-norm solution through the SVD of lhs, singular values at or
    below eps * max(M, N) * s_max dropped. Also returns s (for cond)."""
    torch = torch_mod()
    u, s, vh = torch.linalg.svd(lhs, full_matrices=False)
    cut = float(np.finfo(np.float64).eps) * max(lhs.shape) * s[0]
    keep = s > cut
    inv = torch.where(keep, 1.0 / torch.where(keep, s, torch.ones_like(s)), torch.zeros_like(s))
    return vh.T @ (inv[:, None] * (u.T @ rhs)), s


def legacy_single_pass(
    data: MatrixOrStream,
    cfg: PcaConfig,
    block_rows: Optional[int] = None,
    cond_warn: float = 1e12,
    *,
    precision: str = "auto",
    device=None,
    return_device: bool = False,
) -> TruncatedSvd:
    """Two-sketch one-pass baseline (algorithms.py:312-392): one traversal
    through the pass kernels with Omega_t = Philox(seed, STREAM_COSKETCH)
    (m x l) as the co-sketch operand gives Y = A Omega (as G) and
    Yt = A^T Omega_t (as H); centering (:353-357); Q = orth(Y), Qt = orth(Yt);
    core = lstsq(Omega_t^T Q, Yt^T Qt) (:361-363) with the conditioning
    warning (:365-372); SVD of the core, U = Q U~, V = Qt V~ (:374-378)."""
    import warnings as _warnings

    from .errors import CapabilityError, ConditioningWarning
    from .linalg import STREAM_COSKETCH
    torch = torch_mod()
    stream = as_row_stream(data)
    m = stream.n_rows
    if m is None:
        raise CapabilityError(
            "legacy_single_pass must know the row count up front to draw its "
            "left test matrix; wrap the source in a counted or sized stream")
    if m == 0:
        raise EmptyStreamError("the stream has no rows")
    cfg.validate_dims(stream.n_cols, m)
    dev = default_device(device)
    n, l = stream.n_cols, cfg.l
    omega = gaussian_matrix_device(n, l, cfg.seed, stream=STREAM_SKETCH, device=dev)
    omega_t = gaussian_matrix_device(m, l, cfg.seed, stream=STREAM_COSKETCH, device=dev)
    sk = run_pass(stream, omega, block_rows=block_rows, precision=precision, device=dev, left=omega_t,
                  shift=cfg.center)
    dtype = sk.dtype
    om = sk.omega_used(on_device=True)
    y, yt, col_sums, rows_seen = _finish_pair(sk)
    if rows_seen == 0:
        raise EmptyStreamError("the stream yielded no rows")
    if rows_seen != m:
        raise CapabilityError(f"stream declared {m} rows but yielded {rows_seen}")
    ot = to_device64(omega_t, dev)
    if dtype == np.float32:  # Omega_t as the pass used it, rounded on the device
        ot = ot.float().double()
    mean = None
    if cfg.center:
        mean = col_sums / m
        y = y - (mean @ om)[None, :]
        yt = yt - torch.outer(mean, ot.sum(dim=0))
    q = qr_unpivoted(y, rank_check=False, device=dev).q
    qt = qr_unpivoted(yt, rank_check=False, device=dev).q
    lhs = ot.T @ q
    core, sv = _lstsq_min_norm(lhs, yt.T @ qt)
    notes: tuple = ()
    cond = float(sv[0] / sv[-1]) if float(sv[-1]) > 0.0 else float("inf")
    if cond > cond_warn:
        msg = (f"co-sketch system is ill-conditioned (cond ~ {cond:.3e}); "
               f"singular values may be inaccurate")
        notes = (msg,)
        _warnings.warn(msg, ConditioningWarning, stacklevel=2)
    small = dense_svd(core)
    u, v = sign_align(q @ small.u[:, :cfg.k], qt @ small.v[:, :cfg.k])
    s = small.s[:cfg.k].clone()
    retained = int(m * l + n * l + n * l + m * l + n)  # y + yt + omega + omega_t + col_sums (:383)
    if not return_device:
        u, s, v = host_copy(u), host_copy(s), host_copy(v)
        mean = host_copy(mean) if mean is not None else None
    return TruncatedSvd(u=u, s=s, v=v, mean=mean, passes=_measured_passes(stream, 1),
                        retained_floats=retained, warnings=notes)


def principal_components(svd: TruncatedSvd) -> list:
    """Columns of V in order (algorithms.py:395-398)."""
    return [np.asarray(svd.v)[:, j].copy() for j in range(svd.v.shape[1])]
