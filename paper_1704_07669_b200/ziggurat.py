"""Constants of numpy's float64 ziggurat ``standard_normal`` — the sampler
behind the reference's seeded Gaussian draw (``gaussian_matrix``,
/root/reference/pkg/src/streampca/linalg.py:46-56: ``Generator(Philox(key=
[seed, stream])).standard_normal``) — recovered by probing numpy itself, so
the device draw (``csrc/omega_rng.cuh``) reproduces it bit for bit.

numpy's sampler (the published Marsaglia-Tsang ziggurat, 256 layers) takes
one raw 64-bit draw r per attempt: idx = r & 0xff, sign = bit 8, rabs =
bits 9..60; x = rabs * w[idx] is returned when rabs < k[idx]; otherwise
layer 0 samples the tail beyond R (x = R - log1p(-u1)/R, accepted when
-2 log1p(-u2) > x'^2) and the other layers accept x when
(f[idx-1] - f[idx]) u + f[idx] < exp(-x^2/2); a rejected attempt restarts
on a fresh draw. The tables w, k, f and R are internal to numpy's C code,
so they are read back through the Philox state API: a Philox state's
``buffer`` holds the next four raw draws, which lets this module feed the
sampler chosen raw values and observe the output and how many draws it
consumed.

* w[idx]: the output for rabs = 1 (exact: 1 * w; u = 0 where the layer has no fast range).
* k[idx]: bisection for the smallest rabs that leaves the fast path.
* R: layer-0 tail with u1 = 0 returns exactly R; 1/R is checked the same way.
* f: f[i] = exp(-x_i^2 / 2) at the layer edges x_i = w[i] 2^52 (f[0] = 1),
  confirmed against numpy's accept / reject decisions at bisected
  boundaries (a wrong value would move them).

The result is cached next to this file (``_ziggurat_f64.npz``) keyed by the
numpy version; ``tables()`` re-derives it when the key differs.
"""

from __future__ import annotations

import ctypes
import ctypes.util
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
CACHE = os.path.join(_HERE, "_ziggurat_f64.npz")
_MASK52 = (1 << 52) - 1
_TABLES = None


class _Probe:
    """Feeds up to four raw draws to numpy's standard_normal (the rest come
    from Philox block counter 1 of key 0)."""

    def __init__(self):
        self.bg = np.random.Philox(key=np.array([0, 0], dtype=np.uint64))
        self.gen = np.random.Generator(self.bg)
        self.base = self.bg.state

    def draw(self, raws):
        st = dict(self.base)
        buf = np.zeros(4, dtype=np.uint64)
        buf[: len(raws)] = np.array([int(v) for v in raws], dtype=np.uint64)
        st["buffer"] = buf
        st["buffer_pos"] = 4 - len(raws) if len(raws) < 4 else 0
        if len(raws) < 4:  # the fed values must be the next ones: shift them to the buffer's end
            buf2 = np.zeros(4, dtype=np.uint64)
            buf2[4 - len(raws):] = buf[: len(raws)]
            st["buffer"] = buf2
        self.bg.state = st
        x = float(self.gen.standard_normal())
        used = self.bg.state["buffer_pos"] - st["buffer_pos"]
        if self.bg.state["state"]["counter"][0] != self.base["state"]["counter"][0]:
            used = -1  # ran past the fed values
        return x, used


def _raw(idx: int, sign: int, rabs: int) -> int:
    return (idx & 0xFF) | ((sign & 1) << 8) | ((rabs & _MASK52) << 9)


def _u_raw(u: float) -> int:
    """raw draw whose next_double is u (u a multiple of 2^-53 in [0, 1))."""
    return int(round(u * 2.0 ** 53)) << 11


def _derive():
    p = _Probe()
    fast_raw = _raw(1, 0, 1)  # a fast-path draw with a known output (w[1])
    w = np.zeros(256)
    k = np.zeros(256, dtype=np.uint64)
    for idx in range(256):  # rabs = 1: fast path, or (k[idx] = 0) accepted by the layer test at u = 0
        x, used = p.draw([_raw(idx, 0, 1), 0, fast_raw, fast_raw])
        assert used in (1, 2), (idx, used)
        w[idx] = x
    for idx in range(256):
        _, used = p.draw([_raw(idx, 0, 0), _u_raw(0.5), fast_raw, fast_raw])
        if used != 1:  # no fast range at all
            k[idx] = np.uint64(0)
            continue
        lo, hi = 0, _MASK52 + 1  # fast at lo; find the first rabs that is not
        x, used = p.draw([_raw(idx, 0, _MASK52), _u_raw(0.5), fast_raw, fast_raw])
        if used == 1:
            k[idx] = np.uint64(_MASK52 + 1)
            continue
        while hi - lo > 1:
            mid = (lo + hi) // 2
            _, used = p.draw([_raw(idx, 0, mid), _u_raw(0.5), fast_raw, fast_raw])
            if used == 1:
                lo = mid
            else:
                hi = mid
        k[idx] = np.uint64(hi)
    # tail constant R: layer 0 beyond the fast range with u1 = 0 (log1p(-0) = -0)
    big = int(k[0])
    big = big if not (big >> 8) & 1 else big + 256  # bit 8 of rabs is the tail's sign
    x, used = p.draw([_raw(0, 0, big), 0, _u_raw(0.75), fast_raw])
    assert used == 3, used
    r_tail = x
    libm = ctypes.CDLL(ctypes.util.find_library("m"))
    libm.log1p.restype = ctypes.c_double
    libm.log1p.argtypes = [ctypes.c_double]
    inv_r = 1.0 / r_tail
    for u in (0.5, 0.25, 0.125 + 2.0 ** -40):
        x, used = p.draw([_raw(0, 0, big), _u_raw(u), _u_raw(1 - 2.0 ** -20), fast_raw])
        assert used == 3, used
        assert x == r_tail + (-inv_r * libm.log1p(-u)), ("1/R", u)
    # f: exp(-x^2/2) at the layer edges, checked against numpy's decisions
    f = np.empty(256)
    f[0] = 1.0
    for i in range(1, 256):
        xe = w[i] * 2.0 ** 52
        f[i] = np.exp(-0.5 * xe * xe)
    _check_f(p, w, k, f, fast_raw)
    return dict(w=w, k=k, f=f, r=np.array([r_tail, inv_r]), numpy=np.array([np.__version__]))


def _check_f(p, w, k, f, fast_raw):
    """Bisect u at which numpy's layer-idx decision flips for a few x; the
    candidate f must give the same decision on both sides of each flip."""
    import math
    for idx in list(range(1, 256, 17)) + [1, 2, 254, 255]:
        for frac in (0.3, 0.7):
            rabs = int(int(k[idx]) + frac * (_MASK52 + 1 - int(k[idx])))
            rabs = min(rabs, _MASK52)
            x = rabs * w[idx]
            e = math.exp(-0.5 * x * x)

            def acc_np(u53):
                _, used = p.draw([_raw(idx, 0, rabs), u53 << 11, fast_raw, fast_raw])
                return used == 2

            def acc_f(u53):
                u = u53 * 2.0 ** -53
                return (f[idx - 1] - f[idx]) * u + f[idx] < e

            lo, hi = 0, (1 << 53) - 1
            if acc_np(lo) == acc_np(hi):
                continue
            a_lo = acc_np(lo)
            while hi - lo > 1:
                mid = (lo + hi) // 2
                if acc_np(mid) == a_lo:
                    lo = mid
                else:
                    hi = mid
            if acc_f(lo) != acc_np(lo) or acc_f(hi) != acc_np(hi):
                raise RuntimeError(f"ziggurat f[{idx}] does not reproduce numpy's decision")


def tables():
    """(w float64[256], k uint64[256], f float64[256], R, 1/R)."""
    global _TABLES
    if _TABLES is None:
        d = None
        if os.path.exists(CACHE):
            z = np.load(CACHE)
            if str(z["numpy"][0]) == np.__version__:
                d = {key: z[key] for key in z.files}
        if d is None:
            d = _derive()
            try:
                np.savez(CACHE, **d)
            except OSError:
                pass
        _TABLES = (np.ascontiguousarray(d["w"], dtype=np.float64), np.ascontiguousarray(d["k"], dtype=np.uint64),
                   np.ascontiguousarray(d["f"], dtype=np.float64), float(d["r"][0]), float(d["r"][1]))
    return _TABLES
