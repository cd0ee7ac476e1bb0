"""Full-size U/S/V parity and the multi-rank path with the real CUDA sketch.

* BASELINE config 2 at its full size (100 000 x 10 000 fp32, k = 50, l = 60):
  our single_pass_pca (A resident in HBM) against the oracle's
  single_pass_pca (algorithms.py:165-204 restated; the oracle is pinned to
  the reference by tests/golden) on the same fp32 A widened to fp64 and the
  same seeded Omega — singular values and the largest principal angles of U
  and V within BASELINE.json's fp32 bar, 1e-4.
* sharded_single_pass_pca (Eq. 10 as a row sum) in two
  processes on cuda:0 with a gloo process group, each rank sketching its
  row shard through libspca, against the single-process run of the whole
  matrix. The two ranks' pass kernels are run one after the other (a barrier
  between them): two persistent kernels of different processes must not be
  left to the GPU's time slicing.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp
from threadpoolctl import threadpool_limits

import oracle as O

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1704_07669_b200 as P  # noqa: E402
from paper_1704_07669_b200 import parallel as PAR  # noqa: E402
from paper_1704_07669_b200 import synth  # noqa: E402


def _rel(x, y):
    x, y = np.asarray(x, np.float64), np.asarray(y, np.float64)
    return float(np.max(np.abs(x - y) / np.abs(y)))


def test_config2_full_size_usv_parity():
    cs = synth.config_shape("cfg2")
    a = synth.config_matrix("cfg2", device="cuda")
    cfg = P.PcaConfig(k=cs["k"], oversample=cs["l"] - cs["k"], seed=1)
    res = P.single_pass_pca(P.DeviceRowStream(a), cfg)
    a_host = a.cpu().numpy()
    del a
    torch.cuda.empty_cache()
    with threadpool_limits(limits=os.cpu_count() or 1):
        u, s, v, *_ = O.oracle_single_pass(a_host, k=cfg.k, oversample=cfg.l - cfg.k, block_size=10,
                                           seed=1, block_rows=4096)
    e_s = _rel(res.s, s)
    e_u = O.subspace_angle(res.u, u)
    e_v = O.subspace_angle(res.v, v)
    assert res.u.shape == (cs["m"], cfg.k) and res.v.shape == (cs["n"], cfg.k)
    assert e_s <= 1e-4 and e_u <= 1e-4 and e_v <= 1e-4, (e_s, e_u, e_v)


def _free_port():
    so = socket.socket()
    so.bind(("127.0.0.1", 0))
    p = so.getsockname()[1]
    so.close()
    return p


def _make(m, n, dtype, offset):
    gen = torch.Generator(device="cuda").manual_seed(11)
    x = torch.randn(m, 40, device="cuda", dtype=torch.float64, generator=gen) / m ** 0.5
    w = torch.randn(40, n, device="cuda", dtype=torch.float64, generator=gen)
    w *= (1.0 / torch.arange(1, 41, device="cuda", dtype=torch.float64))[:, None]
    a = x @ w + 1e-3 * torch.randn(m, n, device="cuda", dtype=torch.float64, generator=gen) + offset
    return a.to(dtype)


def _worker(rank, world, port, m, n, dtype_name, center, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1704_07669_b200 import sketch as SK
        inner = SK.sketch_pass

        def one_at_a_time(*a, **kw):  # the ranks' pass kernels never overlap in time
            st = None
            for r in range(world):
                if r == rank:
                    st = inner(*a, **kw)
                    torch.cuda.synchronize()
                dist.barrier()
            return st

        SK.sketch_pass = one_at_a_time
        dtype = getattr(torch, dtype_name)
        a = _make(m, n, dtype, 0.05 if center else 0.0)
        r0, r1 = PAR.shard_rows(m, world, rank)
        cfg = P.PcaConfig(k=12, oversample=8, block_size=10, seed=3, center=center)
        res = PAR.sharded_single_pass_pca(a[r0:r1].contiguous(), cfg, dist)
        torch.cuda.synchronize()
        if rank == 0:
            np.savez(out, u=res.u, s=res.s, v=res.v, retained=res.retained_floats,
                     mean=res.mean if res.mean is not None else np.zeros(0))
    finally:
        dist.destroy_process_group()


# fp64: the only difference is the order of the row sums (two shards added in
# fp64 vs one running sum), 1e-12; the centered case subtracts the mean's
# rank-one sketch after the sum, which amplifies that reorder noise by
# |mean| / spread, 1e-11. fp32: shard-local fp32 accumulators, 1e-5.
@pytest.mark.parametrize("dtype_name,center,tol", [("float64", False, 1e-12), ("float64", True, 1e-11),
                                                    ("float32", False, 1e-5)])
def test_sharded_pca_two_processes_real_sketch(tmp_path, dtype_name, center, tol):
    m, n = 30011, 1500
    out = str(tmp_path / "r.npz")
    mp.spawn(_worker, args=(2, _free_port(), m, n, dtype_name, center, out), nprocs=2, join=True)
    got = np.load(out)
    a = _make(m, n, getattr(torch, dtype_name), 0.05 if center else 0.0)
    cfg = P.PcaConfig(k=12, oversample=8, block_size=10, seed=3, center=center)
    want = P.single_pass_pca(P.DeviceRowStream(a), cfg)
    assert _rel(got["s"], want.s) <= tol
    assert O.subspace_angle(got["u"], want.u) <= tol
    assert O.subspace_angle(got["v"], want.v) <= tol
    assert int(got["retained"]) == want.retained_floats
    if center:
        assert np.max(np.abs(got["mean"] - want.mean)) <= 1e-12
