"""Host logic of the post-pass pieces added for the GPU drivers, run with CPU
torch tensors (no device): CholeskyQR2 against Householder with the
reference's sign convention (linalg.py:71-98), its ill-conditioned fallback,
and the minimum-norm solve that stands in for np.linalg.lstsq
(algorithms.py:363)."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from paper_1704_07669_b200 import linalg as L  # noqa: E402
from paper_1704_07669_b200.algorithms import _lstsq_min_norm  # noqa: E402


def _matrix(m, b, cond, seed):
    g = torch.Generator().manual_seed(seed)
    u, _ = torch.linalg.qr(torch.randn(m, b, dtype=torch.float64, generator=g))
    v, _ = torch.linalg.qr(torch.randn(b, b, dtype=torch.float64, generator=g))
    s = torch.logspace(0, -np.log10(cond), b, dtype=torch.float64)
    return (u * s) @ v.T


@pytest.mark.parametrize("cond", [1.0, 1e2, 1e4])
def test_cholesky_qr2_matches_householder(cond):
    y = _matrix(5000, 10, cond, seed=int(cond))
    q, r = L._cholesky_qr2(y)
    q0, r0 = np.linalg.qr(y.numpy())
    sign = np.where(np.diag(r0) < 0, -1.0, 1.0)
    q0, r0 = q0 * sign, r0 * sign[:, None]
    assert np.abs(q.numpy() - q0).max() < 1e-11 * cond
    assert np.abs(r.numpy() - r0).max() < 1e-13 * np.abs(r0).max()
    assert (np.diag(r.numpy()) > 0).all()
    assert np.abs(q.numpy().T @ q.numpy() - np.eye(10)).max() < 1e-14


@pytest.mark.parametrize("cond", [1e7, 1e13])
def test_cholesky_qr2_falls_back_when_ill_conditioned(cond):
    assert L._cholesky_qr2(_matrix(5000, 10, cond, seed=3)) is None
    y = _matrix(5000, 10, cond, seed=3)
    y[:, 4] = 0.0  # an exactly dependent column
    assert L._cholesky_qr2(y) is None


@pytest.mark.parametrize("rank", [12, 7])
def test_min_norm_solve_matches_numpy_lstsq(rank):
    rng = np.random.default_rng(rank)
    lhs = rng.standard_normal((12, rank)) @ rng.standard_normal((rank, 12))
    rhs = rng.standard_normal((12, 5))
    x, s = _lstsq_min_norm(torch.from_numpy(lhs), torch.from_numpy(rhs))
    ref = np.linalg.lstsq(lhs, rhs, rcond=None)[0]
    assert np.allclose(x.numpy(), ref, rtol=1e-8, atol=1e-10)
    assert np.allclose(s.numpy(), np.linalg.svd(lhs, compute_uv=False))
