"""The fused post-pass (csrc/postpass.cuh, spca_qb_block) against the
reference's blocked_qb restated by the oracle (qb.py:59-171) and against the
library-GEMM form of the same optimistic factorization."""

import numpy as np
import pytest
import torch

import oracle as O

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_1704_07669_b200 import qb as QB  # noqa: E402


def _sketch(m, n, l, seed, rank=None, noise=1e-3):
    rng = np.random.default_rng(seed)
    r = rank or min(m, n)
    a = (rng.standard_normal((m, r)) / np.sqrt(m)) @ (np.diag(1.0 / np.arange(1, r + 1)) @
                                                     rng.standard_normal((r, n)) / np.sqrt(n))
    a += noise * rng.standard_normal((m, n))
    om = rng.standard_normal((n, l))
    g = a @ om
    h = a.T @ g
    return g, h, om


def _rel(x, y):
    return float(torch.linalg.norm(x - y) / torch.linalg.norm(y))


@pytest.mark.parametrize("m,n,l,b", [(4000, 300, 60, 10), (20000, 500, 120, 10), (3000, 900, 250, 10),
                                     (5000, 400, 64, 16), (6000, 300, 36, 6), (6000, 300, 35, 5), (2000, 700, 500, 10), (70000, 300, 120, 10), (9000, 900, 250, 10)])
def test_fused_qb_matches_library_form_and_oracle(m, n, l, b):
    g, h, om = _sketch(m, n, l, seed=m + l)
    dev = torch.device("cuda")
    gt, ht, ot = (torch.from_numpy(x).to(dev) for x in (g, h, om))
    lib = QB._blocked_qb_optimistic(gt, ht, ot, b, dev)
    if b % 2 or l > 256:  # outside spca_qb_block's shapes: the library-GEMM form
        fused = QB.blocked_qb(gt, ht, ot, b)
    else:
        fused = QB._blocked_qb_fused(gt, ht, ot, b, dev)
    assert fused is not None and lib is not None
    assert _rel(fused.q, lib.q) < 1e-11 and _rel(fused.b, lib.b) < 1e-11
    ref = O.oracle_qb(g, h, om, b)
    q_ref = torch.from_numpy(ref.q).to(dev)
    b_ref = torch.from_numpy(ref.b).to(dev)
    assert _rel(fused.q, q_ref) < 1e-10 and _rel(fused.b, b_ref) < 1e-10
    # orthonormal columns
    eye = torch.eye(l, dtype=torch.float64, device=dev)
    assert float((fused.q.T @ fused.q - eye).abs().max()) < 1e-12


def test_fused_qb_bitwise_repeatable():
    g, h, om = _sketch(30000, 400, 120, seed=3)
    dev = torch.device("cuda")
    gt, ht, ot = (torch.from_numpy(x).to(dev) for x in (g, h, om))
    f1 = QB._blocked_qb_fused(gt, ht, ot, 10, dev)
    f2 = QB._blocked_qb_fused(gt, ht, ot, 10, dev)
    assert torch.equal(f1.q, f2.q) and torch.equal(f1.b, f2.b)


def test_fused_qb_flags_deficient_block_and_general_path_repairs(golden):
    """A block with a numerically dependent column leaves the fused path
    (flag set) and blocked_qb falls back to the repair of qb.py:138-171."""
    g, h, om = _sketch(3000, 200, 40, seed=9, rank=25, noise=0.0)  # exact rank 25 < l
    dev = torch.device("cuda")
    gt, ht, ot = (torch.from_numpy(x).to(dev) for x in (g, h, om))
    assert QB._blocked_qb_fused(gt, ht, ot, 10, dev) is None
    res = QB.blocked_qb(gt, ht, ot, 10, on_deficiency="repair", repair_seed=4)
    ref = O.oracle_qb(g, h, om, 10, on_deficiency="repair", repair_seed=4)
    assert res.repaired_columns == tuple(ref.repaired_columns)
    approx = res.q @ res.b
    want = torch.from_numpy(ref.q @ ref.b).to(dev)
    assert _rel(approx, want) < 1e-9


def test_fused_qb_ill_conditioned_blocks_two_pass_path():
    """Blocks with cond(y) ~ 1e3 (columns of G scaled over three decades
    within every block) exceed the one-pass CholeskyQR bound (cond_F <= 16)
    and run both CholeskyQR passes on the device; the result still matches
    the reference's blocked_qb (oracle) at 1e-10 and Q stays orthonormal."""
    g, h, om = _sketch(20000, 400, 60, seed=11)
    scale = np.tile(np.logspace(0, -3, 10), 6)
    g = g * scale[None, :]
    h = h * scale[None, :]
    om = om * scale[None, :]
    dev = torch.device("cuda")
    gt, ht, ot = (torch.from_numpy(x).to(dev) for x in (g, h, om))
    fused = QB._blocked_qb_fused(gt, ht, ot, 10, dev)
    assert fused is not None
    ref = O.oracle_qb(g, h, om, 10)
    assert _rel(fused.q, torch.from_numpy(ref.q).to(dev)) < 1e-10
    assert _rel(fused.b, torch.from_numpy(ref.b).to(dev)) < 1e-10
    eye = torch.eye(60, dtype=torch.float64, device=dev)
    assert float((fused.q.T @ fused.q - eye).abs().max()) < 1e-12
