"""Pin the oracle's restatements of basic_rand_svd (algorithms.py:207-263)
and legacy_single_pass (algorithms.py:312-392) against the real reference's
outputs (tests/golden/golden_alg.npz). CPU only: the oracle is then the
checker of the GPU versions in test_gpu_alg.py."""

import numpy as np
import pytest

import oracle as O
from conftest import ALG_CASES


def _case(golden_alg, name):
    k, p, b, seed, center, br = (int(x) for x in golden_alg[f"{name}_cfg"])
    a = golden_alg[f"{name}_a"].astype(np.float64)
    return a, dict(k=k, oversample=p, block_size=b, seed=seed, center=bool(center), block_rows=br)


@pytest.mark.parametrize("name", ALG_CASES)
def test_basic_rand_svd_bitwise(golden_alg, name):
    a, kw = _case(golden_alg, name)
    u, s, v, mean, q, bm, om = O.oracle_basic_rand_svd(a, **kw)
    assert np.array_equal(s, golden_alg[f"{name}_basic_s"])
    assert np.array_equal(u, golden_alg[f"{name}_basic_u"])
    assert np.array_equal(v, golden_alg[f"{name}_basic_v"])
    if kw["center"]:
        assert np.array_equal(mean, golden_alg[f"{name}_basic_mean"])
    # retained_floats = g + omega + b + col_sums (algorithms.py:262)
    m, n = a.shape
    l = om.shape[1]
    assert golden_alg[f"{name}_basic_meta"].tolist() == [2, m * l + n * l + l * n + n]


@pytest.mark.parametrize("name", ALG_CASES)
def test_legacy_single_pass_bitwise(golden_alg, name):
    a, kw = _case(golden_alg, name)
    u, s, v, mean, cond, y, yt = O.oracle_legacy_single_pass(a, **kw)
    assert np.array_equal(s, golden_alg[f"{name}_legacy_s"])
    assert np.array_equal(u, golden_alg[f"{name}_legacy_u"])
    assert np.array_equal(v, golden_alg[f"{name}_legacy_v"])
    if kw["center"]:
        assert np.array_equal(mean, golden_alg[f"{name}_legacy_mean"])
    m, n = a.shape
    l = y.shape[1]
    # passes, retained = y + yt + omega + omega_t + col_sums (algorithms.py:383), no warning
    assert golden_alg[f"{name}_legacy_meta"].tolist() == [1, m * l + n * l + n * l + m * l + n, 0]
    assert cond < 1e12


def test_legacy_conditioning_warning(golden_alg):
    a = golden_alg["ill_a"]
    _, s, _, _, cond, _, _ = O.oracle_legacy_single_pass(a, k=5, oversample=15, block_size=5, seed=7,
                                                         block_rows=40)
    assert np.array_equal(s, golden_alg["ill_legacy_s"])
    assert cond > 2.0
    assert golden_alg["ill_legacy_nwarn"].tolist() == [1, 1]
    assert f"cond ~ {cond:.3e}" in str(golden_alg["ill_legacy_msg"])
