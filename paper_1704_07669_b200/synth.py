"""Seeded synthetic inputs of the BASELINE.json configs, generated on the GPU.

BASELINE configs 2-5 are A = X diag(s) Y^T + sigma * N(0,1) with
X ~ N(0,1)/sqrt(m) (m x r) and Y ~ N(0,1)/sqrt(n) (n x r), stored fp32.
The reference has no such generator; this one is
block-deterministic: rows [4096 b, 4096 (b+1)) depend only on (seed, b), so
any row shard (multi-GPU) or any host block (config 4's pinned stream) can
be produced independently and reproducibly. No public dataset is involved.
"""

from __future__ import annotations

import math

from .device import default_device, torch_mod

BLOCK = 4096

# name: (m, n, rank, spectrum, noise, k, l)
CONFIGS = {
    # BASELINE config 1 (the reference's CPU-runnable case, fp64): A = U diag(s) V^T,
    # U, V orthonormal from Philox draws, s_i = 10^(-4 (i-1) / 999)
    "cfg1": (2_000, 1_000, 1_000, "log4", 0.0, 20, 30),
    "cfg2": (100_000, 10_000, 200, "inv", 1e-3, 50, 60),
    "cfg3": (1_000_000, 4_096, 300, "exp30", 1e-3, 100, 120),
    "cfg4": (5_000_000, 10_000, 100, "invsqrt", 1e-2, 50, 60),
    "cfg5": (50_000, 200_000, 500, "pow15", 1e-3, 200, 250),
}


def spectrum(kind: str, r: int, device):
    torch = torch_mod()
    i = torch.arange(1, r + 1, dtype=torch.float64, device=device)
    if kind == "inv":
        s = 1.0 / i
    elif kind == "exp30":
        s = torch.exp(-i / 30.0)
    elif kind == "pow15":
        s = i ** -1.5
    elif kind == "invsqrt":
        s = 1.0 / torch.sqrt(i)
    else:
        raise ValueError(kind)
    return s


def _gen(device, seed: int, stream: int):
    torch = torch_mod()
    g = torch.Generator(device=device)
    g.manual_seed((int(seed) * 1_000_003 + int(stream) * 7_919 + 17) % (2 ** 63 - 1))
    return g


def right_factor(n: int, r: int, kind: str, seed: int, device):
    """diag(s) Y^T as an r x n fp32 tensor (shared by every row block)."""
    torch = torch_mod()
    y = torch.randn(n, r, generator=_gen(device, seed, -1), device=device, dtype=torch.float32)
    y /= math.sqrt(n)
    s = spectrum(kind, r, device).to(torch.float32)
    return (y * s).T.contiguous()


def fill_rows(out, r0: int, m: int, n: int, r: int, noise: float, seed: int, w):
    """Write rows [r0, r0 + out.shape[0]) of A into ``out`` (fp32, on w's device),
    block by block, each block from its own seed."""
    torch = torch_mod()
    dev = w.device
    rows = out.shape[0]
    b0 = r0 // BLOCK
    b1 = (r0 + rows - 1) // BLOCK
    for b in range(b0, b1 + 1):
        lo, hi = b * BLOCK, min((b + 1) * BLOCK, m)
        g = _gen(dev, seed, b)
        x = torch.randn(hi - lo, r, generator=g, device=dev, dtype=torch.float32) / math.sqrt(m)
        blk = x @ w
        blk += noise * torch.randn(hi - lo, n, generator=g, device=dev, dtype=torch.float32)
        s0, s1 = max(lo, r0), min(hi, r0 + rows)
        out[s0 - r0:s1 - r0].copy_(blk[s0 - lo:s1 - lo], non_blocking=True)
    return out


def reference_style_matrix(m: int, n: int, seed: int = 100, device=None):
    """BASELINE config 1 on the GPU in fp64: the reference's synth_matrix
    construction (synthetic.py:141-164) — U = Q(Philox(seed, 2) m x r),
    V = Q(Philox(seed, 3) n x r) with diag(R) >= 0, A = U diag(s) V^T,
    s_i = 10^(-4 (i-1) / (r-1)), r = min(m, n). Same draws as the reference
    (linalg.gaussian_matrix); the product is formed by one GEMM instead of the
    reference's row-by-row gemv, so A agrees to rounding, not bitwise (the
    bit-exact matrix is the oracle's, used by the parity tests)."""
    torch = torch_mod()
    from .linalg import STREAM_FACTOR_U, STREAM_FACTOR_V, gaussian_matrix
    dev = default_device(device)
    r = min(m, n)

    def orth(x):
        q, rr = torch.linalg.qr(torch.from_numpy(x).to(dev), mode="reduced")
        return q * torch.where(torch.diagonal(rr) < 0, -1.0, 1.0).to(q.dtype)

    u = orth(gaussian_matrix(m, r, seed, stream=STREAM_FACTOR_U))
    v = orth(gaussian_matrix(n, r, seed, stream=STREAM_FACTOR_V))
    s = 10.0 ** (-4.0 * torch.arange(r, dtype=torch.float64, device=dev) / max(1, r - 1))
    return (u * s) @ v.T


def config_matrix(name: str, device=None, rows=None, seed: int = 2024, m_override=None):
    """A (or rows [r0, r1) of A) of a BASELINE config on the GPU: fp32 for
    configs 2-5, fp64 for config 1."""
    torch = torch_mod()
    dev = default_device(device)
    if name == "cfg1":
        a = reference_style_matrix(CONFIGS["cfg1"][0] if m_override is None else int(m_override),
                                   CONFIGS["cfg1"][1], device=dev)
        return a if rows is None else a[rows[0]:rows[1]].contiguous()
    m, n, r, kind, noise, _, _ = CONFIGS[name]
    if m_override is not None:
        m = int(m_override)
    r0, r1 = (0, m) if rows is None else rows
    w = right_factor(n, r, kind, seed, dev)
    out = torch.empty((r1 - r0, n), dtype=torch.float32, device=dev)
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    try:
        fill_rows(out, r0, m, n, r, noise, seed, w)
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev
    return out


def config_shape(name: str):
    m, n, r, kind, noise, k, l = CONFIGS[name]
    return dict(m=m, n=n, rank=r, spectrum=kind, noise=noise, k=k, l=l)
