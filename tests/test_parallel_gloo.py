"""Multi-rank host logic of the row-sharded pass on CPU (gloo, world size 2).

Each rank sketches its contiguous row shard (the oracle stands in for the
device kernels here), then the production helpers in
paper_1704_07669_b200.parallel combine the shards: one all-reduce of
[H | col_sums | rows], the sharded centering with global statistics, and
the G gather. The combined result must equal the single-process sketch of
the whole matrix (Eq. 10 is a sum over rows).
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from paper_1704_07669_b200 import parallel as PAR


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, m, n, l, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        a = O.gaussian(m, n, seed=5) + 0.75
        om = O.gaussian(n, l, seed=6)
        r0, r1 = PAR.shard_rows(m, world, rank)
        st = O.oracle_sketch(O.row_blocks(a[r0:r1], 7), om)
        h = torch.from_numpy(st.h.copy())
        cs = torch.from_numpy(st.col_sums.copy())
        total = PAR.allreduce_sketch(h, cs, dist, rows=st.rows_seen)
        g_local = torch.from_numpy(st.g.copy())
        g_full, counts = PAR.gather_rows(g_local, dist)
        gc, hc, csc, mu = PAR.center_sharded(g_local, h.clone(), cs.clone(), torch.from_numpy(om),
                                             total, dist)
        gc_full, _ = PAR.gather_rows(gc, dist)
        if rank == 0:
            np.savez(out, h=h.numpy(), cs=cs.numpy(), total=total, g=g_full.numpy(),
                     counts=np.array(counts), gc=gc_full.numpy(), hc=hc.numpy(), mu=mu.numpy(),
                     csc=csc.numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("m", [41, 64])
def test_two_rank_sketch_matches_single_process(tmp_path, m):
    n, l, world = 23, 6, 2
    out = str(tmp_path / "r.npz")
    mp.spawn(_worker, args=(world, _free_port(), m, n, l, out), nprocs=world, join=True)
    r = np.load(out)
    a = O.gaussian(m, n, seed=5) + 0.75
    om = O.gaussian(n, l, seed=6)
    ref = O.oracle_sketch(O.row_blocks(a, 7), om)
    assert int(r["total"]) == m
    assert list(r["counts"]) == [PAR.shard_rows(m, world, k)[1] - PAR.shard_rows(m, world, k)[0]
                                 for k in range(world)]
    assert np.allclose(r["h"], ref.h, rtol=1e-12, atol=1e-12)
    assert np.allclose(r["cs"], ref.col_sums, rtol=1e-12, atol=1e-12)
    assert np.allclose(r["g"], ref.g, rtol=1e-13, atol=1e-13)
    cref = O.oracle_center(ref, om)
    assert np.allclose(r["gc"], cref.g, rtol=1e-10, atol=1e-10)
    assert np.allclose(r["hc"], cref.h, rtol=1e-10, atol=1e-10)
    assert np.allclose(r["mu"], ref.col_sums / m, rtol=1e-12, atol=1e-14)
    assert not r["csc"].any()


def test_shard_rows_partition():
    for m in (1, 7, 100, 101):
        for world in (1, 2, 3, 8):
            spans = [PAR.shard_rows(m, world, k) for k in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == m
            assert all(spans[k][1] == spans[k + 1][0] for k in range(world - 1))
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1
