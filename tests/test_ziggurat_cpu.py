"""The constants the device Omega draw uses (paper_1704_07669_b200/ziggurat.py,
recovered by probing numpy) reproduce numpy's float64 ziggurat
standard_normal bit for bit — the sampler behind the reference's
gaussian_matrix (/root/reference/pkg/src/streampca/linalg.py:46-56). The
restatement below walks the raw Philox stream exactly as csrc/omega_rng.cuh
does (fast path, layer test, tail with libm's log1p / exp via math) and must
match Generator(Philox(key=[seed, stream])).standard_normal on every value,
including the rare layer and tail values."""

import math

import numpy as np
import pytest

from paper_1704_07669_b200 import ziggurat as Z

MASK52 = (1 << 52) - 1


def restated(seed, stream, count):
    w, k, f, r_tail, inv_r = Z.tables()
    w = [float(x) for x in w]
    k = [int(x) for x in k]
    f = [float(x) for x in f]
    raw = [int(x) for x in np.random.Philox(key=np.array([seed, stream], dtype=np.uint64)).random_raw(
        int(count * 1.05) + 1000)]

    def nd(v):
        return (v >> 11) * (1.0 / 9007199254740992.0)

    out, pos, kinds = [], 0, [0, 0, 0]
    while len(out) < count:
        while True:
            r = raw[pos]
            pos += 1
            idx, rr = r & 0xFF, r >> 8
            rabs = (rr >> 1) & MASK52
            x = rabs * w[idx]
            if rr & 1:
                x = -x
            if rabs < k[idx]:
                out.append(x)
                kinds[0] += 1
                break
            if idx == 0:
                while True:
                    xx = -inv_r * math.log1p(-nd(raw[pos]))
                    yy = -math.log1p(-nd(raw[pos + 1]))
                    pos += 2
                    if yy + yy > xx * xx:
                        out.append(-(r_tail + xx) if (rabs >> 8) & 1 else r_tail + xx)
                        break
                kinds[2] += 1
                break
            u = nd(raw[pos])
            pos += 1
            if (f[idx - 1] - f[idx]) * u + f[idx] < math.exp(-0.5 * x * x):
                out.append(x)
                kinds[1] += 1
                break
    return np.array(out[:count]), kinds, pos


@pytest.mark.parametrize("seed,stream", [(1, 0), (7, 1), (0, 4)])
def test_ziggurat_restatement_is_numpy(seed, stream):
    n = 120_000
    got, kinds, _ = restated(seed, stream, n)
    ref = np.random.Generator(np.random.Philox(key=np.array([seed, stream], dtype=np.uint64))).standard_normal(n)
    assert np.array_equal(got, ref)
    assert kinds[1] > 100 and kinds[2] > 5  # the layer and tail paths were exercised


def test_tables_shape_and_cache():
    w, k, f, r_tail, inv_r = Z.tables()
    assert w.shape == (256,) and k.shape == (256,) and f.shape == (256,)
    assert k.dtype == np.uint64 and int(k[1]) == 0  # layer 1 has no fast range
    assert 3.6 < r_tail < 3.7 and inv_r == 1.0 / r_tail
    assert f[0] == 1.0 and np.all(np.diff(f) < 0)
