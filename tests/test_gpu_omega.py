"""The device Omega draw (spca_gaussian_device, csrc/omega_rng.cuh) is the
reference's gaussian_matrix (/root/reference/pkg/src/streampca/linalg.py:46-56:
Generator(Philox(key=[seed, stream])).standard_normal) bit for bit: against
numpy on every BASELINE config's Omega (config 5's 50 M values included, with
their layer and tail values), odd counts, several seeds and streams, and the
Omega hashes recorded from the reference (golden.npz)."""

import ctypes
import hashlib

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_1704_07669_b200 import _lib  # noqa: E402
from paper_1704_07669_b200 import linalg as L  # noqa: E402
from paper_1704_07669_b200.ziggurat import tables  # noqa: E402


def numpy_draw(rows, cols, seed, stream):
    key = np.array([seed, stream], dtype=np.uint64)
    return np.random.Generator(np.random.Philox(key=key)).standard_normal((rows, cols))


def device_draw_rc(count, seed, stream):
    """the raw C-ABI call (no host fallback): return code and values"""
    out = torch.empty(count, dtype=torch.float64, device="cuda")
    w, k, f, r, ir = tables()
    vp = ctypes.c_void_p
    rc = _lib.load().spca_gaussian_device(vp(out.data_ptr()), count, seed, stream, w.ctypes.data_as(vp),
                                          k.ctypes.data_as(vp), f.ctypes.data_as(vp), r, ir,
                                          vp(torch.cuda.current_stream().cuda_stream or 1))
    torch.cuda.synchronize()
    return rc, out.cpu().numpy()


@pytest.mark.parametrize("rows,cols,seed,stream", [
    (1000, 30, 1, 0), (10_000, 60, 1, 0), (4_096, 120, 1, 0), (200_000, 250, 1, 0),
    (1, 1, 3, 0), (7, 1, 0, 2), (1_000_003, 3, 7, 1), (2_000, 1_000, 100, 3), (333, 77, 2, 4),
])
def test_device_draw_bitwise(rows, cols, seed, stream):
    rc, got = device_draw_rc(rows * cols, seed, stream)
    assert rc == _lib.OK  # the device vouched for every value (no host fallback)
    assert np.array_equal(got.reshape(rows, cols), numpy_draw(rows, cols, seed, stream))


def test_public_entry_point_and_reference_hashes(golden):
    _, meta = golden
    for name, n, l in [("cfg1", 1000, 30), ("cfg2", 10000, 60), ("cfg3", 4096, 120)]:
        for seed in (0, 1):
            om = L.gaussian_matrix_device(n, l, seed).cpu().numpy()
            assert hashlib.sha256(np.ascontiguousarray(om).tobytes()).hexdigest()[:16] == \
                meta[f"omega_{name}_s{seed}_f64"]


def test_many_seeds_small():
    for seed in range(20):
        rc, got = device_draw_rc(50_000, seed, seed % 5)
        assert rc == _lib.OK and np.array_equal(got, numpy_draw(50_000, 1, seed, seed % 5).ravel())
