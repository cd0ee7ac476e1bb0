"""The product's Omega draw (linalg.gaussian_matrix, multi-threaded) is the
reference's Philox(seed, stream).standard_normal bit for bit (linalg.py:39-56):
against the serial numpy draw and the Omega hashes recorded from the reference
itself (golden.npz)."""

import hashlib

import numpy as np
import pytest

from paper_1704_07669_b200 import linalg as L


def serial(rows, cols, seed, stream):
    key = np.array([seed, stream], dtype=np.uint64)
    return np.random.Generator(np.random.Philox(key=key)).standard_normal((rows, cols))


@pytest.mark.parametrize("rows,cols,seed,stream", [
    (10_000, 60, 1, 0), (1_000_003, 5, 7, 1), (4_096, 120, 0, 0), (2_000_000, 3, 2, 4), (999, 1000, 3, 0),
])
def test_parallel_draw_bitwise(rows, cols, seed, stream):
    assert np.array_equal(L.gaussian_matrix(rows, cols, seed, stream), serial(rows, cols, seed, stream))


@pytest.mark.parametrize("threads", [2, 3, 8, 16])
def test_parallel_draw_any_thread_count(threads):
    key = np.array([5, 0], dtype=np.uint64)
    n = 3_000_017
    out = L._parallel_normals(key, n, threads)
    assert out is not None and np.array_equal(out, serial(n, 1, 5, 0).ravel())


def test_omega_hashes_match_reference(golden):
    _, meta = golden
    for name, n, l in [("cfg1", 1000, 30), ("cfg2", 10000, 60), ("cfg3", 4096, 120)]:
        for seed in (0, 1):
            om = L.gaussian_matrix(n, l, seed)
            assert hashlib.sha256(np.ascontiguousarray(om).tobytes()).hexdigest()[:16] == \
                meta[f"omega_{name}_s{seed}_f64"]
