"""§8(f) rank 4 on the GPU: the co-sketch operand (spca_sketch_set_left) and
the two algorithms built on it — basic_rand_svd (algorithms.py:207-263) and
legacy_single_pass (algorithms.py:312-392) — against the oracle and the
reference's own outputs (golden_alg.npz). Bars as BASELINE.json: fp64 1e-10
on singular values and principal angles (1e-12 on raw sketches), fp32 1e-4."""

import warnings

import numpy as np
import pytest

import oracle as O
from conftest import ALG_CASES

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs CUDA", allow_module_level=True)

import paper_1704_07669_b200 as P  # noqa: E402


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def _tc_ok():
    try:
        P.GpuSketch(64, np.ones((64, 16)), np.float32, precision="tc").close()
        return True
    except Exception:
        return False


def _precisions(dtype):
    if dtype == np.float64:
        return ["auto"]
    return ["simt", "tc"] if _tc_ok() else ["simt"]


# ------------------------------------------------------------ co-sketch pass
@pytest.mark.parametrize("dtype,precision,m,n,l", [
    (np.float64, "simt", 700, 90, 12),
    (np.float32, "simt", 3000, 500, 40),
    (np.float32, "tc", 5000, 1000, 60),
    (np.float32, "tc", 3000, 4096, 120),
    (np.float32, "tc", 2100, 2000, 250),
])
def test_cosketch_vs_oracle(dtype, precision, m, n, l):
    """H = A^T L with L the co-sketch operand; G = A Omega and col_sums as usual."""
    if precision == "tc" and not _tc_ok():
        pytest.skip("no tensor-core path")
    a = O.gaussian(m, n, seed=m + 1).astype(dtype)
    om = O.gaussian(n, l, seed=n + 2)
    left = O.gaussian(m, l, seed=l + 3)
    sk = P.GpuSketch(n, om, dtype, precision=precision)
    sk.set_left(left)
    sk.push(a, 0, final=True)
    g, h, cs, rows = sk.finish(on_device=False)
    sk.close()
    a64 = a.astype(np.float64)
    used = (lambda x: x.astype(np.float32).astype(np.float64)) if dtype == np.float32 else (lambda x: x)
    tol = 1e-12 if dtype == np.float64 else 2e-5
    assert rows == m
    assert rel(g, a64 @ used(om)) <= tol
    assert rel(h, a64.T @ used(left)) <= tol
    assert np.allclose(cs, a64.sum(axis=0), rtol=1e-5, atol=1e-4)


def test_cosketch_block_independent_and_reset():
    """Any push split gives bitwise the same H; reset keeps L; set_left(None)
    restores the plain sketch."""
    if not _tc_ok():
        pytest.skip("no tensor-core path")
    m, n, l = 9000, 700, 60
    a = O.gaussian(m, n, seed=8).astype(np.float32)
    om, left = O.gaussian(n, l, seed=9), O.gaussian(m, l, seed=10)
    sk = P.GpuSketch(n, om, np.float32, precision="tc")
    sk.set_left(left)
    sk.push(a, 0, final=True)
    _, h1, _, _ = sk.finish(on_device=False)
    sk.reset()
    for r0 in range(0, m, 1777):
        sk.push(a[r0:r0 + 1777], r0)
    _, h2, _, _ = sk.finish(on_device=False)
    assert np.array_equal(h1, h2)
    sk.reset()
    sk.set_left(None)
    sk.push(a, 0, final=True)
    g3, h3, _, _ = sk.finish(on_device=False)
    sk.close()
    assert rel(h3, a.astype(np.float64).T @ g3) <= 2e-5


def test_cosketch_too_many_rows_and_state():
    sk = P.GpuSketch(20, O.gaussian(20, 4, seed=1), np.float64)
    sk.set_left(O.gaussian(10, 4, seed=2))
    with pytest.raises(P.CapabilityError):
        sk.push(O.gaussian(11, 20, seed=3), 0)
    sk.reset()
    sk.push(O.gaussian(5, 20, seed=3), 0)
    with pytest.raises(P.StreamPcaError):
        sk.set_left(O.gaussian(10, 4, seed=2))  # after the first push of a pass
    sk.close()


@pytest.mark.parametrize("precision", ["tc", "simt"])
def test_cosketch_normalized(precision):
    """Co-sketch of normalize_rows(A) (fused normalisation on the TC path:
    operand L / norm and the finish-time correction with L)."""
    if precision == "tc" and not _tc_ok():
        pytest.skip("no tensor-core path")
    m, n, l = 4000, 1000, 60
    rng = np.random.default_rng(3)
    a = (O.gaussian(m, n, seed=4) * rng.uniform(0.1, 10, (m, 1)) + rng.normal(0, 30, (m, 1))).astype(np.float32)
    a[5] = 1.5
    om, left = O.gaussian(n, l, seed=5), O.gaussian(m, l, seed=6)
    sk = P.GpuSketch(n, om, np.float32, precision=precision, normalize=True)
    sk.set_left(left)
    sk.push(a, 0, final=True)
    g, h, cs, _ = sk.finish(on_device=False)
    sk.close()
    an = O.oracle_normalize_rows(a.astype(np.float64))
    l32 = left.astype(np.float32).astype(np.float64)
    assert rel(h, an.T @ l32) <= 2e-5, rel(h, an.T @ l32)
    assert rel(g, an @ om.astype(np.float32).astype(np.float64)) <= 2e-5


# ------------------------------------------------- basic / legacy end to end
def _case(golden_alg, name):
    k, p, b, seed, center, br = (int(x) for x in golden_alg[f"{name}_cfg"])
    a = golden_alg[f"{name}_a"]
    return a, P.PcaConfig(k=k, oversample=p, block_size=b, seed=seed, center=bool(center)), br


def _check(res, golden_alg, name, algo, tol):
    s_ref = golden_alg[f"{name}_{algo}_s"]
    assert float(np.max(np.abs(res.s - s_ref) / s_ref)) <= tol
    # principal angles of the leading (well separated) components
    kk = res.s.shape[0]
    assert O.subspace_angle(res.u[:, :kk], golden_alg[f"{name}_{algo}_u"][:, :kk]) <= tol * 100
    assert O.subspace_angle(res.v[:, :kk], golden_alg[f"{name}_{algo}_v"][:, :kk]) <= tol * 100
    if res.mean is not None:
        assert np.allclose(res.mean, golden_alg[f"{name}_{algo}_mean"], rtol=1e-6, atol=1e-9)


@pytest.mark.parametrize("name", ALG_CASES)
def test_basic_rand_svd_vs_reference(golden_alg, name):
    a, cfg, br = _case(golden_alg, name)
    for prec in _precisions(a.dtype):
        res = P.basic_rand_svd(a, cfg, block_rows=br, precision=prec)
        tol = 1e-10 if a.dtype == np.float64 else 1e-4
        s_ref = golden_alg[f"{name}_basic_s"]
        assert float(np.max(np.abs(res.s - s_ref) / s_ref)) <= tol, prec
        if a.dtype == np.float64:  # vectors: 1e-10 on the directions (sign-aligned, so elementwise)
            assert np.abs(res.u - golden_alg[f"{name}_basic_u"]).max() <= 1e-8
            assert np.abs(res.v - golden_alg[f"{name}_basic_v"]).max() <= 1e-8
        else:
            _check(res, golden_alg, name, "basic", tol)
        assert res.passes == 2
        assert res.retained_floats == int(golden_alg[f"{name}_basic_meta"][1])


@pytest.mark.parametrize("name", ALG_CASES)
def test_legacy_single_pass_vs_reference(golden_alg, name):
    a, cfg, br = _case(golden_alg, name)
    for prec in _precisions(a.dtype):
        with warnings.catch_warnings():
            warnings.simplefilter("error")  # no conditioning warning on these cases
            res = P.legacy_single_pass(a, cfg, block_rows=br, precision=prec)
        tol = 1e-10 if a.dtype == np.float64 else 1e-4
        s_ref = golden_alg[f"{name}_legacy_s"]
        assert float(np.max(np.abs(res.s - s_ref) / s_ref)) <= tol, prec
        if a.dtype == np.float64:
            assert np.abs(res.u - golden_alg[f"{name}_legacy_u"]).max() <= 1e-8
            assert np.abs(res.v - golden_alg[f"{name}_legacy_v"]).max() <= 1e-8
        else:
            _check(res, golden_alg, name, "legacy", tol)
        assert res.passes == 1 and res.warnings == ()
        assert res.retained_floats == int(golden_alg[f"{name}_legacy_meta"][1])


def test_legacy_conditioning_warning(golden_alg):
    a = golden_alg["ill_a"]
    cfg = P.PcaConfig(k=5, oversample=15, block_size=5, seed=7)
    with pytest.warns(P.ConditioningWarning, match="co-sketch system is ill-conditioned"):
        res = P.legacy_single_pass(a, cfg, block_rows=40, cond_warn=2.0)
    assert len(res.warnings) == 1
    s_ref = golden_alg["ill_legacy_s"]
    assert np.allclose(res.s, s_ref, rtol=1e-10)
    # the condition number the message reports matches the reference's to 4 digits
    assert str(golden_alg["ill_legacy_msg"]).split("cond ~ ")[1][:5] == res.warnings[0].split("cond ~ ")[1][:5]


def test_legacy_row_count_contract():
    a = O.gaussian(50, 12, seed=1)
    cfg = P.PcaConfig(k=2, oversample=2, block_size=2)

    class Lying(P.ArrayRowStream):  # declares fewer rows than it yields
        @property
        def n_rows(self):
            return 40
    with pytest.raises(P.CapabilityError):
        P.legacy_single_pass(Lying(a), cfg)

    class Short(P.ArrayRowStream):  # declares more rows than it yields
        @property
        def n_rows(self):
            return 60
    with pytest.raises(P.CapabilityError, match="declared 60 rows but yielded 50"):
        P.legacy_single_pass(Short(a), cfg)


def test_streams_through_basic_and_legacy(tmp_path):
    """File, device and generator sources give the in-memory results."""
    a = O.synth_lowrank_plus_noise(3000, 500, 40, "inv", 1e-3, seed=12)
    cfg = P.PcaConfig(k=10, seed=2)
    ref_b = P.basic_rand_svd(a, cfg)
    ref_l = P.legacy_single_pass(a, cfg)
    path = str(tmp_path / "a.spca")
    P.matfile.write_matrix(path, a, dtype="float32", header=True)
    dev = torch.from_numpy(a).cuda()
    for src in [P.DeviceRowStream(dev), P.PassCounter(P.ArrayRowStream(a)), P.FileRowStream(path)]:
        rb = P.basic_rand_svd(src, cfg)
        assert np.array_equal(rb.s, ref_b.s)
    rl = P.legacy_single_pass(P.DeviceRowStream(dev), cfg)
    assert np.array_equal(rl.s, ref_l.s)
    pc = P.PassCounter(P.ArrayRowStream(a))
    assert P.basic_rand_svd(pc, cfg).passes == 2


def test_basic_matches_single_pass_config2_shape():
    """Full config-2 shape (100 000 x 10 000 fp32 on the device): the two-pass
    yardstick and the single-pass estimate agree on the leading singular
    values (the reference: 'identical seeds give singular values agreeing
    to rounding' for exactly low-rank data; here to the sketch's accuracy)."""
    from paper_1704_07669_b200 import synth
    a = synth.config_matrix("cfg2", device="cuda")
    cfg = P.PcaConfig(k=50, oversample=10, seed=1)
    rb = P.basic_rand_svd(P.DeviceRowStream(a), cfg)
    rs = P.single_pass_pca(P.DeviceRowStream(a), cfg)
    rl = P.legacy_single_pass(P.DeviceRowStream(a), cfg)
    assert np.all(np.isfinite(rb.s)) and np.all(np.isfinite(rl.s))
    top = 10  # signal components, well above the noise bulk
    assert np.max(np.abs(rb.s[:top] - rs.s[:top]) / rs.s[:top]) <= 2e-2
    assert O.subspace_angle(rb.v[:, :5], rs.v[:, :5]) <= 5e-2
    del a
    torch.cuda.empty_cache()


# ------------------------------------------------------------ column shift
def _offset_data(m, n, seed, offset=0.75):
    """BASELINE-style fp32 data on a large common mean (offset ~300x the spread):
    the case where post-hoc centering cancels fp32 accumulator rounding."""
    return (O.synth_lowrank_plus_noise(m, n, 40, "exp30", 1e-3, seed=seed) + offset).astype(np.float32)


@pytest.mark.parametrize("precision,left", [("tc", False), ("tc", True), ("simt", False), ("simt", True)])
def test_shift_sketch_vs_oracle(precision, left):
    """spca_sketch_set_shift: same G, H, col_sums as the unshifted sketch (the
    shift is undone in fp64), and the centered sketch accurate to fp32 of the
    data's spread rather than of its mean."""
    if precision == "tc" and not _tc_ok():
        pytest.skip("no tensor-core path")
    m, n, l = 6000, 800, 60
    a = _offset_data(m, n, seed=31)
    om = O.gaussian(n, l, seed=32)
    lm = O.gaussian(m, l, seed=33) if left else None
    sk = P.GpuSketch(n, om, np.float32, precision=precision, shift=True)
    if left:
        sk.set_left(lm)
    for r0 in range(0, m, 2500):  # several pushes: c is the pass's first row
        sk.push(a[r0:r0 + 2500], r0)
    g, h, cs, _ = sk.finish(on_device=False)
    sk.close()
    a64 = a.astype(np.float64)
    om32 = om.astype(np.float32).astype(np.float64)
    opnd = lm.astype(np.float32).astype(np.float64) if left else None
    g_ref = a64 @ om32
    h_ref = a64.T @ (opnd if left else g_ref)
    assert rel(g, g_ref) <= 1e-6 and rel(h, h_ref) <= 1e-6
    assert np.allclose(cs, a64.sum(axis=0), rtol=1e-9)
    # centered: G_c = G - 1 mu^T Omega; H_c = H - mu 1^T(G or L)
    mu = a64.mean(axis=0)
    ac = a64 - mu
    gc = g - (mu @ om32)[None, :]
    hc = h - np.outer(mu, (opnd if left else g).sum(axis=0))
    assert rel(gc, ac @ om32) <= 2e-5, rel(gc, ac @ om32)
    hc_ref = ac.T @ (opnd if left else ac @ om32)
    assert rel(hc, hc_ref) <= 2e-5, rel(hc, hc_ref)


@pytest.mark.parametrize("dtype,precision,m,n,l", [
    (np.float32, "tc", 2100, 2000, 250),   # column groups of 128
    (np.float32, "tc", 3000, 4096, 120),   # l_pad = 128
    (np.float32, "tc", 1500, 1000, 60),    # n not a multiple of 32 (2-D A loads)
    (np.float64, "auto", 900, 300, 20),    # DFMA path
])
def test_shift_shapes(dtype, precision, m, n, l):
    if precision == "tc" and not _tc_ok():
        pytest.skip("no tensor-core path")
    rng = np.random.default_rng(n)
    a = (O.gaussian(m, n, seed=m) * 1e-2 + rng.normal(0, 5, size=(1, n))).astype(dtype)
    om = O.gaussian(n, l, seed=l)
    st = P.sketch_pass(P.ArrayRowStream(a), om, precision=precision, shift=True)
    a64 = a.astype(np.float64)
    om_u = om.astype(np.float32).astype(np.float64) if dtype == np.float32 else om
    assert np.array_equal(st.omega, om_u)  # spca_omega_used: exactly the values the pass used
    g_ref = a64 @ om_u
    tol = 1e-6 if dtype == np.float32 else 1e-12
    assert rel(st.g, g_ref) <= tol and rel(st.h, a64.T @ g_ref) <= tol
    # centered sketches: accurate to the data's spread, not its (500x larger)
    # mean. (fp64: the post-hoc centering below — the reference's own
    # center_correct, in fp64 — itself loses ~u (mean/spread)^2 sqrt(n) ~ 1e-9.)
    mu = a64.mean(axis=0)
    gc = st.g - (mu @ om_u)[None, :]
    hc = st.h - np.outer(mu, st.g.sum(axis=0))
    ac = a64 - mu
    assert rel(gc, ac @ om_u) <= (2e-5 if dtype == np.float32 else 1e-10)
    assert rel(hc, ac.T @ (ac @ om_u)) <= (2e-5 if dtype == np.float32 else 1e-8)


def test_shift_bitwise_splits_and_errors():
    if not _tc_ok():
        pytest.skip("no tensor-core path")
    a = _offset_data(7000, 600, seed=34)
    om = O.gaussian(600, 60, seed=35)
    st1 = P.sketch_pass(P.ArrayRowStream(a), om, shift=True)
    st2 = P.sketch_pass(P.ArrayRowStream(a), om, block_rows=999, shift=True)
    assert np.array_equal(st1.g, st2.g) and np.array_equal(st1.h, st2.h)
    assert np.array_equal(st1.col_sums, st2.col_sums)
    bad = a.copy()
    bad[0, 5] = np.nan  # the shift row itself is non-finite: still DataError(row=0)
    with pytest.raises(P.DataError) as ei:
        P.sketch_pass(P.ArrayRowStream(bad), om, shift=True)
    assert ei.value.row == 0
    bad = a.copy()
    bad[4321, 7] = np.inf
    with pytest.raises(P.DataError) as ei:
        P.sketch_pass(P.ArrayRowStream(bad), om, shift=True)
    assert ei.value.row == 4321
    sk = P.GpuSketch(600, om, np.float32, normalize=True)
    with pytest.raises(P.ConfigError):  # shift and normalisation are exclusive
        sk.set_shift(True)
    sk.close()


def _oracle_power_refine(a, k, seed, oversample=10, block_size=10, block_rows=4096):
    """power_refine (algorithms.py:266-309) composed from the oracle's pieces,
    centered: sketch, center, Omega2 = orth(H), sketch, center, blocked QB."""
    a = a.astype(np.float64)
    l = O.sketch_width(k, oversample, block_size)
    om = O.gaussian(a.shape[1], l, seed)
    st = O.oracle_center(O.oracle_sketch(O.row_blocks(a, block_rows), om), om)
    om2, _ = O.qr_pos(st.h, rank_check=False)
    st2 = O.oracle_center(O.oracle_sketch(O.row_blocks(a, block_rows), om2), om2)
    qb = O.oracle_qb(st2.g, st2.h, om2, block_size, on_deficiency="repair", repair_seed=seed)
    sv = O.thin_svd(qb.b)
    u, v = O.align_signs(qb.q @ sv.u[:, :k], sv.v[:, :k])
    return sv.s[:k], v


@pytest.mark.parametrize("algo", ["single", "basic", "legacy", "power"])
def test_centered_fp32_offset_data(algo):
    """Centered PCA of fp32 data on a large mean matches the fp64 oracle on
    the same fp32 values within the fp32 bar (1e-4) on every device path."""
    a = _offset_data(5000, 700, seed=36)
    cfg = P.PcaConfig(k=15, seed=3, center=True, power=1 if algo == "power" else 0)
    for prec in _precisions(np.float32):
        if algo == "single":
            res = P.single_pass_pca(a, cfg, precision=prec)
            _, s_ref, v_ref, *_ = O.oracle_single_pass(a, k=15, seed=3, center=True, block_rows=4096)
        elif algo == "basic":
            res = P.basic_rand_svd(a, cfg, precision=prec)
            _, s_ref, v_ref, *_ = O.oracle_basic_rand_svd(a, k=15, seed=3, center=True)
        elif algo == "legacy":
            res = P.legacy_single_pass(a, cfg, precision=prec)
            _, s_ref, v_ref, *_ = O.oracle_legacy_single_pass(a, k=15, seed=3, center=True)
        else:
            res = P.power_refine(a, cfg, precision=prec)
            s_ref, v_ref = _oracle_power_refine(a, k=15, seed=3)
        err = float(np.max(np.abs(res.s - s_ref) / s_ref))
        assert err <= 1e-4, (prec, err)
        assert O.subspace_angle(res.v[:, :5], v_ref[:, :5]) <= 1e-3, prec


# ------------------------------------------------- spca_allreduce (C ABI, NCCL)
def _nccl_single_rank_comm():
    """A one-rank NCCL communicator on the current GPU through ctypes (what a
    C/C++ host would hold); None when libnccl is not loadable."""
    import ctypes
    try:
        nccl = ctypes.CDLL("libnccl.so.2", mode=ctypes.RTLD_GLOBAL)
    except OSError:
        return None, None
    class UniqueId(ctypes.Structure):  # ncclUniqueId, passed by value
        _fields_ = [("internal", ctypes.c_char * 128)]

    uid = UniqueId()
    assert nccl.ncclGetUniqueId(ctypes.byref(uid)) == 0
    comm = ctypes.c_void_p()
    nccl.ncclCommInitRank.argtypes = [ctypes.POINTER(ctypes.c_void_p), ctypes.c_int, UniqueId, ctypes.c_int]
    assert nccl.ncclCommInitRank(ctypes.byref(comm), 1, uid, 0) == 0
    return nccl, comm


def test_spca_allreduce_single_rank():
    """The C-ABI exchange step on a one-rank communicator: [H | col_sums] and G
    unchanged bitwise, the global row count returned; state errors."""
    torch.cuda.set_device(0)
    nccl, comm = _nccl_single_rank_comm()
    if nccl is None:
        pytest.skip("libnccl.so.2 not loadable")
    a = O.gaussian(3000, 500, seed=41).astype(np.float32)
    om = O.gaussian(500, 40, seed=42)
    sk = P.GpuSketch(500, om, np.float32)
    sk.push(a, 0, final=True)
    with pytest.raises(P.StreamPcaError):
        sk.allreduce_nccl(comm.value)  # before finish
    g, h, cs, m = sk.finish(on_device=False)
    assert sk.allreduce_nccl(comm.value) == 3000
    g2, h2, cs2, m2 = sk.finish(on_device=False)
    assert np.array_equal(h, h2) and np.array_equal(cs, cs2) and np.array_equal(g, g2) and m2 == m
    sk.close()
    nccl.ncclCommDestroy(comm)


# ------------------------------------------------------------- wide sketches
@pytest.mark.parametrize("dtype,precision,m,n,l", [
    (np.float32, "tc", 2000, 1500, 300),    # three column groups of 128
    (np.float32, "tc", 1500, 2048, 700),    # six groups, l_pad 768
    (np.float32, "simt", 1200, 900, 330),
    (np.float64, "auto", 900, 800, 310),    # DMMA, five 64-column l tiles
])
def test_wide_sketch_vs_oracle(dtype, precision, m, n, l):
    """Sketch widths beyond 256 (k + oversample of a few hundred): the
    reference accepts any l <= min(m, n)."""
    if precision == "tc" and not _tc_ok():
        pytest.skip("no tensor-core path")
    a = O.gaussian(m, n, seed=l).astype(dtype)
    om = O.gaussian(n, l, seed=l + 1)
    st = P.sketch_pass(P.ArrayRowStream(a), om, precision=precision)
    om_u = om.astype(np.float32).astype(np.float64) if dtype == np.float32 else om
    ref = O.oracle_sketch(O.row_blocks(a.astype(np.float64), 4096), om_u)
    tol = 2e-5 if dtype == np.float32 else 1e-12
    assert rel(st.g, ref.g) <= tol and rel(st.h, ref.h) <= tol


def test_wide_pca_k300():
    """single_pass_pca with k = 300 (l = 310) on fp32 data: the 1e-4 bar."""
    a = O.synth_lowrank_plus_noise(3000, 1200, 400, "exp30", 1e-3, seed=9)
    res = P.single_pass_pca(a, P.PcaConfig(k=300, seed=1))
    _, s_ref, v_ref, *_ = O.oracle_single_pass(a, k=300, seed=1, block_rows=4096)
    assert float(np.max(np.abs(res.s[:100] - s_ref[:100]) / s_ref[:100])) <= 1e-4


# ------------------------------------------- any n on the tensor-core path
@pytest.mark.parametrize("n", [1001, 333, 4098])
def test_tc_row_stride_not_16_bytes(n, tmp_path):
    """Row strides that TMA cannot address (n % 4 != 0, or an unaligned view)
    are re-strided through a padded buffer: same sketch as the oracle from
    device, pinned, pageable and file sources, bitwise equal across them, and
    with normalisation, column shift and a co-sketch operand."""
    if not _tc_ok():
        pytest.skip("no tensor-core path")
    m, l = 5000, 60
    a = (O.gaussian(m, n, seed=n) + 0.5).astype(np.float32)
    om = O.gaussian(n, l, seed=n + 1)
    om32 = om.astype(np.float32).astype(np.float64)
    ref = O.oracle_sketch(O.row_blocks(a.astype(np.float64), 4096), om32)
    st = P.sketch_pass(P.ArrayRowStream(a), om, precision="tc")
    assert rel(st.g, ref.g) <= 2e-5 and rel(st.h, ref.h) <= 2e-5
    dev = torch.from_numpy(a).cuda()
    pin = torch.from_numpy(a).pin_memory()
    path = str(tmp_path / "a.spca")
    P.matfile.write_matrix(path, a, dtype="float32", header=True)
    for src in [P.DeviceRowStream(dev), P.PinnedRowStream(pin), P.FileRowStream(path)]:
        s2 = P.sketch_pass(src, om, precision="tc")
        assert np.array_equal(np.asarray(s2.g), st.g) and np.array_equal(np.asarray(s2.h), st.h)
    # an unaligned device view (column offset 1): stride n + 1, base not 16-byte aligned
    wide = torch.zeros((m, n + 1), dtype=torch.float32, device="cuda")
    wide[:, 1:] = dev
    s3 = P.sketch_pass(P.DeviceRowStream(wide[:, 1:]), om, precision="tc")
    assert np.array_equal(np.asarray(s3.h), st.h)
    # normalisation, shift and co-sketch through the padded path
    sn = P.sketch_pass(P.NormalizedRowStream(P.ArrayRowStream(a)), om, precision="tc")
    rn = O.oracle_sketch(O.row_blocks(O.oracle_normalize_rows(a.astype(np.float64)), 4096), om32)
    assert rel(sn.h, rn.h) <= 2e-5
    ss = P.sketch_pass(P.ArrayRowStream(a), om, precision="tc", shift=True)
    assert rel(ss.h, ref.h) <= 1e-6
    left = O.gaussian(m, l, seed=3)
    sk = P.GpuSketch(n, om, np.float32, precision="tc")
    sk.set_left(left)
    sk.push(a, 0, final=True)
    _, hl, _, _ = sk.finish(on_device=False)
    sk.close()
    assert rel(hl, a.astype(np.float64).T @ left.astype(np.float32).astype(np.float64)) <= 2e-5


def test_config1_device_construction_matches_reference(golden):
    """bench.py's config-1 matrix (the reference's synth_matrix construction
    from the same Philox draws, built on the device) gives the reference's
    config-1 singular values (golden.npz, reference run) within the fp64 bar."""
    from paper_1704_07669_b200 import synth
    g, _ = golden
    a = synth.config_matrix("cfg1", device="cuda")
    assert a.dtype == torch.float64 and tuple(a.shape) == (2000, 1000)
    res = P.single_pass_pca(P.DeviceRowStream(a), P.PcaConfig(k=20, oversample=10, block_size=10, seed=1),
                            block_rows=200)
    s_ref = g["cfg1_s"]
    assert float(np.max(np.abs(res.s - s_ref) / s_ref)) <= 1e-10


def test_two_handles_on_two_streams():
    """Pass kernels of different handles on different streams are ordered on
    the device (a persistent kernel needs every SM): pushes interleaved on two
    streams complete and equal the single-handle results."""
    if not _tc_ok():
        pytest.skip("no tensor-core path")
    m, n, l = 60000, 4000, 60
    a = torch.randn((m, n), device="cuda", dtype=torch.float32, generator=torch.Generator("cuda").manual_seed(5))
    b = torch.randn((m, n), device="cuda", dtype=torch.float32, generator=torch.Generator("cuda").manual_seed(6))
    om = O.gaussian(n, l, seed=7)
    ref_a = P.GpuSketch(n, om, np.float32, precision="tc")
    ref_a.push(a, 0, final=True)
    ga, ha, _, _ = ref_a.finish()
    ref_a.close()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    torch.cuda.synchronize()
    k1 = P.GpuSketch(n, om, np.float32, precision="tc", stream=s1)
    k2 = P.GpuSketch(n, om, np.float32, precision="tc", stream=s2)
    for _ in range(3):  # enqueue both before either completes
        k1.reset()
        k2.reset()
        k1.push(a, 0, final=True)
        k2.push(b, 0, final=True)
        g1, h1, _, _ = k1.finish()
        g2, h2, _, _ = k2.finish()
        assert torch.equal(h1, ha) and torch.equal(g1, ga)
        assert torch.isfinite(h2).all()
    k1.close()
    k2.close()


@pytest.mark.gpu
def test_pass_beside_foreign_kernels():
    """The persistent pass kernel is launched cooperatively (every CTA
    co-scheduled): with foreign work holding SMs on other streams — a
    long-running spin kernel and a stream of torch GEMMs — the pass still
    completes and equals the undisturbed result bit for bit."""
    if not _tc_ok():
        pytest.skip("no tensor-core path")
    m, n, l = 40000, 3000, 60
    a = torch.randn((m, n), device="cuda", dtype=torch.float32, generator=torch.Generator("cuda").manual_seed(8))
    om = O.gaussian(n, l, seed=9)
    ref = P.GpuSketch(n, om, np.float32, precision="tc")
    ref.push(a, 0, final=True)
    g0, h0, c0, _ = ref.finish()
    ref.close()
    s_spin, s_gemm, s_pass = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
    x = torch.randn((2048, 2048), device="cuda")
    torch.cuda.synchronize()
    k = P.GpuSketch(n, om, np.float32, precision="tc", stream=s_pass)
    for _ in range(2):
        with torch.cuda.stream(s_spin):
            torch.cuda._sleep(50_000_000)  # ~25 ms on one SM
        with torch.cuda.stream(s_gemm):
            for _ in range(20):
                x = (x @ x).clamp_(-1, 1)
        k.reset()
        k.push(a, 0, final=True)
        g1, h1, c1, _ = k.finish()
        assert torch.equal(h1, h0) and torch.equal(g1, g0) and torch.equal(c1, c0)
    torch.cuda.synchronize()
    k.close()


@pytest.mark.gpu
@pytest.mark.parametrize("m,n,l", [(1089, 2080, 60), (257, 1000, 30), (2081, 4000, 120), (3000 + 33, 999 * 4, 60)])
def test_padded_k_blocks_read_zero_fill_not_memory(m, n, l):
    """Partial K blocks (n or the row count not a multiple of 32) and, in builds
    with paired MMA-warp iterations (SPCA_BUILD_KPAIR: an odd tail of 32-deep K
    blocks takes one more block, csrc/sketch_fused.cuh fused_decode), whole extra
    blocks must come from TMA out-of-bounds zero fill: the matrix here is a view
    into a larger buffer whose other columns and rows are NaN, so a block that
    read memory beyond n or beyond the last row would poison G or H.
    Odd K-block counts over n (G units) and over the rows (H units)."""
    torch = pytest.importorskip("torch")
    if not _tc_ok():
        pytest.skip("tensor-core path unavailable")
    ld = (n + 64 + 3) // 4 * 4  # 16-byte row stride, at least 64 spare columns
    big = torch.full((m + 96, ld), float("nan"), dtype=torch.float32, device="cuda")
    a = O.gaussian(m, n, seed=m + 1).astype(np.float32)
    big[:m, :n] = torch.from_numpy(a).cuda()
    om = O.gaussian(n, l, seed=n + 1)
    st = P.sketch_pass(P.DeviceRowStream(big[:m, :n]), om, precision="tc")
    assert np.isfinite(st.g).all() and np.isfinite(st.h).all() and np.isfinite(st.col_sums).all()
    ref = O.oracle_sketch(O.row_blocks(a, 4096), om.astype(np.float32).astype(np.float64))
    assert rel(st.g, ref.g) <= 2e-5 and rel(st.h, ref.h) <= 2e-5
    # the same rows pushed in two pieces (a partial chunk in the middle of the stream)
    s2 = P.sketch_pass(P.DeviceRowStream(big[:m, :n]), om, precision="tc", block_rows=m // 2 + 1)
    assert np.array_equal(st.g, s2.g) and np.array_equal(st.h, s2.h)
