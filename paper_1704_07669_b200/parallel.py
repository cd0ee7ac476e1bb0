"""Row-sharded multi-GPU sketch (one process per GPU, torch.distributed/NCCL).

The pass shards by rows with no exchange: G_i depends only on A_i and Omega
(Eq. 10). The single exchange step is the sum of the
per-rank partial sketches: one all-reduce of the packed [H | col_sums |
rows] buffer, n*(l+1)+1 float64 values, issued on the compute stream right
after the last chunk. G stays row-sharded; the post-pass
gathers it to every rank (G is m x l, small next to A).

All functions take plain tensors plus a process group, so the host logic is
exercised with ``gloo`` on CPU tensors in the tests and with ``nccl`` on
CUDA tensors in production.
"""

from __future__ import annotations

from typing import Optional

from .device import host_copy, torch_mod


def _host_staged(dist, group, t) -> bool:
    """gloo has no all_gather on CUDA tensors: such collectives go through
    host copies (NCCL takes the device tensors as they are)."""
    return bool(getattr(t, "is_cuda", False)) and dist.get_backend(group) == "gloo"


def allreduce_sketch(h, col_sums, dist, rows: Optional[int] = None, group=None):
    """Sum H (n x l) and col_sums (n) over ranks in place with ONE collective;
    returns the global row count when ``rows`` is given."""
    torch = torch_mod()
    n, l = h.shape
    extra = 1 if rows is not None else 0
    buf = torch.empty(n * (l + 1) + extra, dtype=torch.float64, device=h.device)
    buf[: n * l].copy_(h.reshape(-1))
    buf[n * l: n * (l + 1)].copy_(col_sums)
    if extra:
        buf[-1] = float(rows)
    if _host_staged(dist, group, buf):
        hb = buf.cpu()
        dist.all_reduce(hb, op=dist.ReduceOp.SUM, group=group)
        buf.copy_(hb)
    else:
        dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=group)
    h.copy_(buf[: n * l].view(n, l))
    col_sums.copy_(buf[n * l: n * (l + 1)])
    return int(round(float(buf[-1]))) if extra else None


def shard_rows(m: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous row range of ``rank`` (first ranks take the remainder)."""
    base, rem = divmod(m, world)
    r0 = rank * base + min(rank, rem)
    return r0, r0 + base + (1 if rank < rem else 0)


def gather_rows(g, dist, group=None):
    """All-gather row shards of different lengths into the full matrix."""
    torch = torch_mod()
    world = dist.get_world_size(group)
    if _host_staged(dist, group, g):
        full, counts = gather_rows(g.cpu(), dist, group)
        return full.to(g.device), counts
    cnt = torch.tensor([g.shape[0]], dtype=torch.int64, device=g.device)
    counts = [torch.zeros_like(cnt) for _ in range(world)]
    dist.all_gather(counts, cnt, group=group)
    counts = [int(c.item()) for c in counts]
    mx = max(counts)
    pad = torch.zeros((mx, g.shape[1]), dtype=g.dtype, device=g.device)
    pad[: g.shape[0]].copy_(g)
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad, group=group)
    return torch.cat([p[:c] for p, c in zip(parts, counts)], dim=0), counts


def center_sharded(g_local, h, col_sums, omega, m_total: int, dist, group=None):
    """center_correct (sketch.py:119-139) with global statistics: mu from the
    all-reduced col_sums, 1^T G summed over every rank's G rows."""
    torch = torch_mod()
    mu = col_sums / m_total
    gsum = g_local.sum(dim=0)
    if _host_staged(dist, group, gsum):
        gh = gsum.cpu()
        dist.all_reduce(gh, op=dist.ReduceOp.SUM, group=group)
        gsum = gh.to(g_local.device)
    else:
        dist.all_reduce(gsum, op=dist.ReduceOp.SUM, group=group)
    g_c = g_local - (mu @ omega)[None, :]
    h_c = h - torch.outer(mu, gsum)
    return g_c, h_c, torch.zeros_like(col_sums), mu


def sharded_single_pass_pca(local_rows, cfg, dist, group=None, precision: str = "auto",
                            on_deficiency: str = "repair", device=None):
    """single_pass_pca over a row-sharded matrix: each rank passes its own
    rows (a CUDA tensor), one all-reduce combines the sketches, every rank
    runs the post-pass on the gathered G and returns the same TruncatedSvd."""
    torch = torch_mod()
    from .algorithms import TruncatedSvd, finish_svd
    from .errors import EmptyStreamError
    from .linalg import STREAM_SKETCH, gaussian_matrix_device
    from .qb import blocked_qb
    from .sketch import sketch_pass
    from .streams import DeviceRowStream

    n = int(local_rows.shape[1])
    omega = gaussian_matrix_device(n, cfg.l, cfg.seed, stream=STREAM_SKETCH, device=device)
    st = sketch_pass(DeviceRowStream(local_rows), omega, precision=precision,
                     device=device, keep_on_device=True, shift=cfg.center)
    h = st.h.clone()
    cs = st.col_sums.clone()
    m_total = allreduce_sketch(h, cs, dist, rows=st.rows_seen, group=group)
    if m_total == 0:
        raise EmptyStreamError("the stream yielded no rows")
    cfg.validate_dims(n, m_total)
    g = st.g
    mean = None
    if cfg.center:
        g, h, cs, mean = center_sharded(g, h, cs, st.omega, m_total, dist, group)
    g_full, _ = gather_rows(g, dist, group)
    factor = blocked_qb(g_full, h, st.omega, cfg.block_size, on_deficiency=on_deficiency,
                        repair_seed=cfg.seed)
    u, s, v = finish_svd(factor, cfg.k)
    retained = int(g_full.numel() + h.numel() + cs.numel() + st.omega.numel())
    return TruncatedSvd(u=host_copy(u), s=host_copy(s), v=host_copy(v),
                        mean=None if mean is None else host_copy(mean), passes=1,
                        retained_floats=retained)
