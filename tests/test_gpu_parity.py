"""CUDA path vs the CPU oracle / golden reference outputs (needs a B200).

Everything here calls through libspca.so (the C ABI) via the Python mirror
of the reference API. Tolerances follow BASELINE.json: fp64 1e-10 relative
on singular values and principal angles (1e-12 on raw sketches, the
reference's own test_sketch.py:35-42 bar); fp32 data 1e-4.
"""

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs CUDA", allow_module_level=True)

import paper_1704_07669_b200 as P  # noqa: E402


def rel(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


PRECISIONS_F32 = ["simt", "tc"]


def _tc_ok():
    try:
        sk = P.GpuSketch(64, np.ones((64, 16)), np.float32, precision="tc")
        sk.close()
        return True
    except Exception:
        return False


# --------------------------------------------------------------- sketch_pass
class TestSketchPass:
    def test_golden_small(self, golden):
        g, _ = golden
        a = O.gaussian(40, 30, seed=3)
        st = P.sketch_pass(P.ArrayRowStream(a), O.gaussian(30, 8, seed=4), block_rows=7)
        assert rel(st.g, g["sk_small_g"]) <= 1e-12
        assert rel(st.h, g["sk_small_h"]) <= 1e-12
        assert np.allclose(st.col_sums, g["sk_small_cs"], rtol=1e-13, atol=1e-13)
        assert st.rows_seen == 40

    def test_identity(self, golden):
        g, _ = golden
        om = O.gaussian(5, 3, seed=1)
        st = P.sketch_pass(P.ArrayRowStream(np.eye(5)), om, block_rows=2)
        assert np.allclose(st.g, om) and np.allclose(st.h, om)
        assert np.allclose(st.col_sums, np.ones(5)) and st.rows_seen == 5

    def test_zero(self):
        st = P.sketch_pass(P.ArrayRowStream(np.zeros((6, 4))), O.gaussian(4, 2, seed=2))
        assert not st.g.any() and not st.h.any() and not st.col_sums.any()

    def test_nonfinite_row_reported(self, golden):
        g, _ = golden
        a = O.gaussian(10, 4, seed=15)
        a[6, 2] = np.inf
        with pytest.raises(P.DataError) as exc:
            P.sketch_pass(P.ArrayRowStream(a), O.gaussian(4, 2, seed=16), block_rows=4)
        assert exc.value.row == int(g["sk_nonfinite_row"]) == 6

    @pytest.mark.parametrize("dtype", [np.float32, np.float64])
    def test_nan_first_row_large(self, dtype):
        a = O.gaussian(5000, 300, seed=1).astype(dtype)
        a[4321, 7] = np.nan
        a[4999, 0] = -np.inf
        with pytest.raises(P.DataError) as exc:
            P.sketch_pass(P.ArrayRowStream(a), O.gaussian(300, 40, seed=2))
        assert exc.value.row == 4321

    def test_width_mismatch(self):
        with pytest.raises(P.StreamFormatError):
            P.sketch_pass(P.ArrayRowStream(np.ones((4, 3))), O.gaussian(5, 2, seed=1))

    def test_bad_block_shape_from_generic_stream(self):
        blocks = [np.ones((3, 4)), np.ones((2, 5))]
        with pytest.raises(P.StreamFormatError):
            P.sketch_pass(P.GeneratorRowStream(iter(blocks), n_cols=4), O.gaussian(4, 2, seed=1))

    def test_default_block_rows_is_sketch_width(self):
        seen = []

        class Probe(P.RowStream):
            def __init__(self, a):
                self.a = a

            n_rows = property(lambda s: s.a.shape[0])
            n_cols = property(lambda s: s.a.shape[1])
            resettable = property(lambda s: True)

            def blocks(self, block_rows):
                seen.append(block_rows)
                for r in range(0, self.a.shape[0], block_rows):
                    yield P.RowBlock(r, self.a[r:r + block_rows])

        P.sketch_pass(Probe(O.gaussian(12, 6, seed=17)), O.gaussian(6, 5, seed=18))
        assert seen == [5]

    def test_memory_accounting(self):
        m, n, l = 30, 20, 6
        st = P.sketch_pass(P.ArrayRowStream(O.gaussian(m, n, seed=19)), O.gaussian(n, l, seed=20))
        assert st.retained_floats == m * l + n * l + n

    def test_single_pass_counted(self):
        pc = P.PassCounter(P.ArrayRowStream(O.gaussian(20, 10, seed=5)))
        P.sketch_pass(pc, O.gaussian(10, 4, seed=6))
        assert pc.passes_completed == 1 and pc.rows_read == 20

    def test_compensated_col_sums(self, golden):
        g, _ = golden
        a = O.gaussian(500, 3, seed=13) + 1e8
        st = P.sketch_pass(P.ArrayRowStream(a), O.gaussian(3, 2, seed=14), compensated=True)
        assert np.allclose(st.col_sums, a.sum(axis=0), rtol=1e-15)
        assert np.allclose(st.col_sums, g["sk_kahan_cs"], rtol=1e-15)

    def test_bitwise_independent_of_block_size(self):
        """Canonical chunking: any push sizes give identical bytes (the GPU
        analogue of acceptance criterion 9, test_acceptance.py:223-255)."""
        a = O.gaussian(9000, 257, seed=9)
        om = O.gaussian(257, 30, seed=10)
        ref = P.sketch_pass(P.ArrayRowStream(a), om)
        for br in (1, 30, 37, 4096, 9000):
            st = P.sketch_pass(P.GeneratorRowStream(iter([a]), n_cols=257), om, block_rows=br)
            assert np.array_equal(st.g, ref.g) and np.array_equal(st.h, ref.h)
            assert np.array_equal(st.col_sums, ref.col_sums)

    def test_run_to_run_bitwise(self):
        a = O.gaussian(7000, 500, seed=21).astype(np.float32)
        om = O.gaussian(500, 60, seed=22)
        r1 = P.sketch_pass(P.ArrayRowStream(a), om)
        r2 = P.sketch_pass(P.ArrayRowStream(a), om)
        assert np.array_equal(r1.g, r2.g) and np.array_equal(r1.h, r2.h)

    @pytest.mark.parametrize("m,n,l", [(1, 1, 1), (3, 7, 2), (129, 65, 33), (1000, 1001, 60),
                                       (4097, 300, 120), (700, 50, 250)])
    def test_fp64_shapes_vs_oracle(self, m, n, l):
        a = O.gaussian(m, n, seed=m + n)
        om = O.gaussian(n, l, seed=l)
        st = P.sketch_pass(P.ArrayRowStream(a), om, block_rows=97)
        ref = O.oracle_sketch(O.row_blocks(a, 97), om)
        assert rel(st.g, ref.g) <= 1e-12 and rel(st.h, ref.h) <= 1e-12
        assert np.allclose(st.col_sums, ref.col_sums, rtol=1e-12, atol=1e-12)

    @pytest.mark.parametrize("precision", PRECISIONS_F32)
    @pytest.mark.parametrize("m,n,l", [(5000, 1000, 60), (3000, 4096, 120), (300, 2000, 250),
                                       (1000, 333, 30), (257, 100, 8), (3000, 1000, 129),
                                       (2100, 4096, 250), (1500, 1000, 384)])
    def test_fp32_shapes_vs_oracle(self, precision, m, n, l):
        if precision == "tc" and not _tc_ok():
            pytest.skip("tensor-core path unavailable")
        a = O.gaussian(m, n, seed=m).astype(np.float32)
        om = O.gaussian(n, l, seed=n)
        try:
            st = P.sketch_pass(P.ArrayRowStream(a), om, precision=precision)
        except P.ConfigError:
            pytest.skip("shape unsupported by this precision")
        om32 = om.astype(np.float32).astype(np.float64)
        ref = O.oracle_sketch(O.row_blocks(a, 4096), om32)
        # fp32-class accumulation over n (G) and m (H) terms; 3xTF32 keeps
        # ~22 significant bits per product (2^-22 ~ 2.4e-7), FFMA 24
        tol = 2e-6 if precision == "simt" else 2e-5
        assert rel(st.g, ref.g) <= tol, rel(st.g, ref.g)
        assert rel(st.h, ref.h) <= tol, rel(st.h, ref.h)
        # column sums: exact fp64 on the SIMT path; the tensor-core pass sums each
        # unit's rows in fp32 (pairwise + Kahan, ~2 ulp of sum|a|) and the units in
        # fp64, i.e. ~1e-7 of the column's absolute sum
        cs_tol = 1e-9 if precision == "simt" else 1e-6
        scale = np.abs(a).astype(np.float64).sum(axis=0)
        assert np.all(np.abs(st.col_sums - ref.col_sums) <= cs_tol * scale + 1e-12)

    def test_device_and_pinned_sources_match_host(self):
        a = O.gaussian(6000, 700, seed=31).astype(np.float32)
        om = O.gaussian(700, 60, seed=32)
        host = P.sketch_pass(P.ArrayRowStream(a), om)
        dev = P.sketch_pass(P.DeviceRowStream(torch.from_numpy(a).cuda()), om)
        pin = P.sketch_pass(P.PinnedRowStream(torch.from_numpy(a).pin_memory()), om)
        for st in (dev, pin):
            assert np.array_equal(st.g, host.g) and np.array_equal(st.h, host.h)

    def test_center_correct_matches_explicit(self, golden):
        g, _ = golden
        a = O.gaussian(50, 40, seed=0) + 2.5
        om = O.gaussian(40, 9, seed=100)
        st = P.center_correct(P.sketch_pass(P.ArrayRowStream(a), om), om)
        assert rel(st.g, g["center_g"]) <= 1e-10 and rel(st.h, g["center_h"]) <= 1e-10
        assert not np.asarray(st.col_sums).any()

    def test_symmetry_of_cross_gram(self):
        a = O.gaussian(25, 12, seed=11)
        om = O.gaussian(12, 5, seed=12)
        st = P.sketch_pass(P.ArrayRowStream(a), om)
        cross = om.T @ st.h
        assert np.linalg.norm(cross - cross.T) <= 1e-10 * np.linalg.norm(cross)


# ------------------------------------------------------------------ blocked_qb
class TestBlockedQb:
    def test_invariants_every_block(self):
        a = O.gaussian(60, 50, seed=1)
        om = O.gaussian(50, 20, seed=2)
        st = P.sketch_pass(P.ArrayRowStream(a), om, keep_on_device=True)
        at = torch.from_numpy(a).cuda()
        seen = []

        def probe(i, q, b):
            seen.append(i)
            assert float((q.T @ q - torch.eye(q.shape[1], device=q.device, dtype=q.dtype)).abs().max()) <= 1e-10
            assert float(torch.linalg.norm(b - q.T @ at)) <= 1e-10 * float(torch.linalg.norm(at))

        f = P.blocked_qb(st.g, st.h, om, 5, on_block=probe)
        assert seen == [0, 1, 2, 3] and not f.repaired_columns

    def test_repair_matches_reference(self, golden):
        g, _ = golden
        u, _ = O.qr_pos(O.gaussian(30, 5, 13, stream=2))
        v, _ = O.qr_pos(O.gaussian(30, 5, 13, stream=3))
        a = u @ (np.linspace(5.0, 1.0, 5)[:, None] * v.T)
        om = O.gaussian(30, 10, 14)
        st = P.sketch_pass(P.ArrayRowStream(a), om, keep_on_device=True)
        f = P.blocked_qb(st.g, st.h, om, 5, on_deficiency="repair")
        assert f.repaired_columns == tuple(g["qb_rep_cols"].tolist())
        q = f.q.cpu().numpy()
        b = f.b.cpu().numpy()
        assert np.max(np.abs(q.T @ q - np.eye(10))) <= 1e-10
        assert np.linalg.norm(a - q @ b) <= 1e-10 * np.linalg.norm(a)
        qr, br = g["qb_rep_q"], g["qb_rep_b"]
        assert np.linalg.norm(q @ b - qr @ br) <= 1e-10 * np.linalg.norm(a)

    def test_deficiency_error_location(self, golden):
        g, _ = golden
        u, _ = O.qr_pos(O.gaussian(30, 5, 13, stream=2))
        v, _ = O.qr_pos(O.gaussian(30, 5, 13, stream=3))
        a = u @ (np.linspace(5.0, 1.0, 5)[:, None] * v.T)
        om = O.gaussian(30, 10, 14)
        st = P.sketch_pass(P.ArrayRowStream(a), om, keep_on_device=True)
        with pytest.raises(P.RankDeficiencyError) as exc:
            P.blocked_qb(st.g, st.h, om, 5)
        assert exc.value.block == int(g["qb_err_block"])
        assert exc.value.column == int(g["qb_err_col"])

    def test_width_not_multiple(self):
        a = O.gaussian(20, 15, seed=11)
        om = O.gaussian(15, 10, seed=12)
        st = P.sketch_pass(P.ArrayRowStream(a), om, keep_on_device=True)
        with pytest.raises(P.ConfigError):
            P.blocked_qb(st.g, st.h, om, 4)


# ------------------------------------------------------------- single_pass_pca
def _assert_svd_close(res, u, s, v, tol):
    s_err = float(np.max(np.abs(res.s - s) / np.abs(s)))
    assert s_err <= tol, f"S rel err {s_err:.2e} > {tol}"
    au = O.subspace_angle(res.u, u)
    av = O.subspace_angle(res.v, v)
    assert au <= tol and av <= tol, f"angles U {au:.2e} V {av:.2e} > {tol}"
    return s_err, au, av


class TestSinglePass:
    def test_config1_parity(self, golden):
        """BASELINE config 1 (fp64): S and subspaces within 1e-10 of the reference."""
        g, _ = golden
        i = np.arange(1, 1001)
        a = O.reference_synth_matrix(2000, 1000, 10.0 ** (-4.0 * (i - 1) / 999.0), seed=100)
        cfg = P.PcaConfig(k=20, oversample=10, block_size=10, seed=1)
        res = P.single_pass_pca(a, cfg, block_rows=200)
        _assert_svd_close(res, g["cfg1_u"], g["cfg1_s"], g["cfg1_v"], 1e-10)
        assert res.passes == 1 and res.retained_floats == int(g["cfg1_retained"])
        # component signs follow the reference convention, so vectors match directly
        assert np.max(np.abs(res.v - g["cfg1_v"])) <= 1e-8

    @pytest.mark.parametrize("precision", PRECISIONS_F32)
    def test_fp32_construction_parity(self, golden, precision):
        if precision == "tc" and not _tc_ok():
            pytest.skip("tensor-core path unavailable")
        g, _ = golden
        a = O.synth_lowrank_plus_noise(4000, 1500, 200, "inv", 1e-3, seed=11)
        res = P.single_pass_pca(a, P.PcaConfig(k=50, oversample=10, seed=1), block_rows=1024,
                                precision=precision)
        _assert_svd_close(res, g["f32_u"], g["f32_s"], g["f32_v"], 1e-4)

    def test_exact_low_rank(self, golden):
        g, _ = golden
        rng = np.random.default_rng(0)
        a = rng.standard_normal((150, 5)) @ rng.standard_normal((5, 100))
        res = P.single_pass_pca(a, P.PcaConfig(k=5, seed=1))
        _assert_svd_close(res, g["spca_lr_u"], g["spca_lr_s"], g["spca_lr_v"], 1e-10)
        with pytest.raises(P.RankDeficiencyError):
            P.single_pass_pca(a, P.PcaConfig(k=5, seed=1), on_deficiency="error")

    def test_centered(self, golden):
        g, _ = golden
        rng = np.random.default_rng(21)
        base = rng.standard_normal((120, 9)) @ rng.standard_normal((9, 60))
        a = base + np.outer(np.ones(120), rng.standard_normal(60))
        res = P.single_pass_pca(a, P.PcaConfig(k=9, center=True))
        _assert_svd_close(res, g["spca_ctr_u"], g["spca_ctr_s"], g["spca_ctr_v"], 1e-10)
        assert np.allclose(res.mean, g["spca_ctr_mean"], rtol=0, atol=1e-12)

    def test_type2_acceptance_input(self, golden):
        g, _ = golden
        sigma = np.arange(1, 501, dtype=np.float64) ** -2.0
        a = O.reference_synth_matrix(500, 500, sigma, seed=100)
        res = P.single_pass_pca(a, P.PcaConfig(k=20, seed=1))
        _assert_svd_close(res, g["type2_u"], g["type2_s"], g["type2_v"], 1e-10)

    def test_generator_stream_unknown_rows(self):
        rng = np.random.default_rng(5)
        a = rng.standard_normal((90, 40))
        res = P.single_pass_pca(P.GeneratorRowStream(iter(a.reshape(9, 10, 40)), n_cols=40),
                                P.PcaConfig(k=5))
        ref = P.single_pass_pca(a, P.PcaConfig(k=5))
        assert np.allclose(res.s, ref.s, rtol=0, atol=1e-12)

    def test_errors_and_accounting(self):
        with pytest.raises(P.EmptyStreamError):
            P.single_pass_pca(np.empty((0, 30)), P.PcaConfig(k=3, oversample=0, block_size=1))
        with pytest.raises(P.ConfigError):
            P.single_pass_pca(np.eye(30), P.PcaConfig(k=3, power=1))
        rng = np.random.default_rng(5)
        a = rng.standard_normal((90, 40))
        pc = P.PassCounter(P.ArrayRowStream(a))
        cfg = P.PcaConfig(k=5, oversample=5)
        res = P.single_pass_pca(pc, cfg)
        assert res.passes == 1 and pc.passes_completed == 1
        assert res.retained_floats == 90 * cfg.l + 2 * 40 * cfg.l + 40

    def test_sign_convention(self):
        res = P.single_pass_pca(np.random.default_rng(11).standard_normal((80, 50)), P.PcaConfig(k=8))
        for j in range(8):
            col = res.v[:, j]
            assert col[np.argmax(np.abs(col))] > 0

    def test_power_refine_matches_oracle_two_pass(self):
        rng = np.random.default_rng(3)
        a = rng.standard_normal((400, 120)) @ np.diag(1.0 / np.arange(1, 121)) @ rng.standard_normal((120, 200))
        res = P.power_refine(a, P.PcaConfig(k=10, power=1, seed=2))
        assert res.passes == 2
        s_true = np.linalg.svd(a, compute_uv=False)[:10]
        assert np.max(np.abs(res.s - s_true) / s_true) < 1e-2


# -------------------------------------------------- full-size properties (cfg2)
def test_config2_full_size_properties():
    """BASELINE config 2 at full size on the device: H = A^T G and G = A Omega
    checked through random probes in fp64 (size-independent properties),
    Omega^T H symmetric, and bitwise reproducibility."""
    from paper_1704_07669_b200 import synth
    a = synth.config_matrix("cfg2", device="cuda")
    m, n = a.shape
    om = O.gaussian(n, 60, 1)
    st = P.sketch_pass(P.DeviceRowStream(a), om, keep_on_device=True)
    om32 = torch.from_numpy(om.astype(np.float32)).cuda().double()
    gen = torch.Generator(device="cuda").manual_seed(0)
    x = torch.randn(60, 4, device="cuda", dtype=torch.float64, generator=gen)
    y = torch.randn(n, 4, device="cuda", dtype=torch.float64, generator=gen)
    a64_rows = a[:20000].double()
    g_ref = a64_rows @ (om32 @ x)
    assert float(torch.linalg.norm(st.g[:20000] @ x - g_ref) / torch.linalg.norm(g_ref)) < 2e-5
    # y^T H x = (A y)^T (G x)
    ay = torch.cat([a[i:i + 20000].double() @ y for i in range(0, m, 20000)])
    lhs = y.T @ st.h @ x
    rhs = ay.T @ (st.g @ x)
    assert float(torch.linalg.norm(lhs - rhs) / torch.linalg.norm(rhs)) < 1e-5
    cross = om32.T @ st.h
    assert float(torch.linalg.norm(cross - cross.T) / torch.linalg.norm(cross)) < 1e-5
    st2 = P.sketch_pass(P.DeviceRowStream(a), om, keep_on_device=True)
    assert torch.equal(st.h, st2.h) and torch.equal(st.g, st2.g)


@pytest.mark.gpu
@pytest.mark.parametrize("precision", ["simt", "tc"])
def test_final_push_matches_push_then_finish(precision):
    """spca_sketch_push_final processes the trailing partial chunk with the
    block: bitwise identical to push + finish, and later pushes are refused."""
    if precision == "tc" and not _tc_ok():
        pytest.skip("tensor-core path unavailable")
    a = torch.from_numpy(O.gaussian(5000, 1200, seed=41).astype(np.float32)).cuda()
    om = O.gaussian(1200, 60, seed=42)
    out = []
    for final in (False, True):
        sk = P.GpuSketch(1200, om, np.float32, precision=precision, rows_hint=5000)
        sk.push(a[:3000], 0)
        sk.push(a[3000:], 3000, final=final)
        if final:
            with pytest.raises(P.DeviceError):
                sk.push(a[:10], 5000)
        g, h, c, rows = sk.finish(on_device=False)
        sk.close()
        out.append((g, h, c, rows))
    assert out[0][3] == out[1][3] == 5000
    for x, y in zip(out[0][:3], out[1][:3]):
        assert np.array_equal(x, y)


# ------------------------------------------------------- disk streaming (§8 f)
@pytest.mark.parametrize("dtype,precision", [("float64", "auto"), ("float32", "simt"), ("float32", "tc")])
@pytest.mark.parametrize("header", [True, False])
def test_file_stream_matches_array(tmp_path, dtype, precision, header):
    """FileRowStream through page-locked buffers == the same rows handed over
    in memory, bitwise (canonical chunking), for several buffer sizes."""
    if precision == "tc" and not _tc_ok():
        pytest.skip("no tensor-core path")
    m, n, l = 5000, 300, 24
    a = O.gaussian(m, n, seed=21).astype(dtype)
    om = O.gaussian(n, l, seed=22)
    p = tmp_path / "a.mat"
    P.matfile.write_matrix(p, a, dtype=dtype, header=header)
    want = P.sketch_pass(P.ArrayRowStream(a), om, precision=precision)
    kw = {} if header else dict(rows=m, cols=n, dtype=dtype)
    for buf in (1 << 20, 333 * n * a.itemsize, 64 << 20):
        fs = P.FileRowStream(p, buffer_bytes=buf, **kw)
        got = P.sketch_pass(fs, om, precision=precision)
        assert got.rows_seen == m
        for x, y in ((got.g, want.g), (got.h, want.h), (got.col_sums, want.col_sums)):
            assert np.array_equal(x, y)
        assert fs.bytes_read == m * n * a.itemsize


def test_file_stream_nonfinite_row_and_pca(tmp_path):
    m, n = 3000, 64
    a = O.gaussian(m, n, seed=23).astype(np.float32)
    a[2222, 5] = np.inf
    p = tmp_path / "bad.spca"
    P.matfile.write_matrix(p, a, dtype="float32")
    with pytest.raises(P.DataError) as ei:
        P.sketch_pass(P.FileRowStream(p, buffer_bytes=200 * n * 4), O.gaussian(n, 8, seed=1))
    assert ei.value.row == 2222
    # end to end through single_pass_pca and the pass counter
    a[2222, 5] = 0.0
    P.matfile.write_matrix(p, a, dtype="float32")
    cfg = P.PcaConfig(k=5, oversample=5, block_size=5, seed=3)
    res_f = P.single_pass_pca(P.FileRowStream(p, buffer_bytes=1 << 20), cfg)
    res_a = P.single_pass_pca(a, cfg)
    assert np.array_equal(res_f.s, res_a.s)
    pc = P.PassCounter(P.FileRowStream(p))
    P.sketch_pass(pc, O.gaussian(n, 8, seed=1))
    assert pc.passes_completed == 1 and pc.rows_read == m


# ------------------------------------- row normalisation + estimator (§8 f)
def test_normalize_rows_kernel(golden_f):
    x = golden_f["norm_in"]
    got = P.normalize_rows(x)
    assert got.dtype == np.float64
    # fp64 with a different summation order than numpy's pairwise sum: ~1 ulp,
    # except row 7 (1e6 offset: the mean's rounding, 1e6 * 2^-52, survives centering)
    err = np.abs(got - golden_f["norm_out"]).max(axis=1)
    assert np.all(np.delete(err, 7) <= 1e-15) and err[7] <= 1e-11
    assert np.array_equal(got[2], np.zeros(13)) and np.array_equal(got[4], np.zeros(13))
    blk = P.normalize_rows(P.RowBlock(17, x))
    assert blk.first_row_index == 17 and np.array_equal(blk.values, got)
    # device tensors stay on the device in their dtype; in place works
    t = torch.from_numpy(x.astype(np.float32)).cuda()
    d = P.normalize_rows(t)
    assert d.is_cuda and d.dtype == torch.float32
    want32 = O.oracle_normalize_rows(x.astype(np.float32).astype(np.float64))
    assert np.abs(d.cpu().numpy() - want32).max() <= 1.2e-7  # fp64 arithmetic, fp32 output
    from paper_1704_07669_b200.sketch import normalize_rows_device
    normalize_rows_device(t, t)
    assert torch.equal(t, d)
    # wide rows (several strides per thread) vs the oracle
    w = O.gaussian(33, 70001, seed=9) + 5.0
    assert np.allclose(P.normalize_rows(w), O.oracle_normalize_rows(w), rtol=0, atol=1e-15)
    # register-resident vector path (n a multiple of the vector width, up to
    # 12288 fp32 / 6144 fp64), with constant and zero rows, out of place and in place
    for dt, width in ((np.float32, 10000), (np.float64, 6144), (np.float32, 12288), (np.float64, 6146)):
        z = O.gaussian(70, width, seed=11) * 2.0 + 3.0
        z[3] = 1.25
        z[5] = 0.0
        zd = torch.from_numpy(z.astype(dt)).cuda()
        want = O.oracle_normalize_rows(z.astype(dt).astype(np.float64))
        got = normalize_rows_device(zd).cpu().numpy().astype(np.float64)
        tol = 1.2e-7 if dt == np.float32 else 1e-15
        assert np.abs(got - want).max() <= tol, (dt, width)
        assert not got[3].any() and not got[5].any()
        normalize_rows_device(zd, zd)
        assert np.array_equal(zd.cpu().numpy().astype(np.float64), got)


@pytest.mark.parametrize("source", ["array", "device", "generator", "file"])
def test_normalized_stream_pca(golden_f, tmp_path, source):
    a = golden_f["ns_a"].astype(np.float64)  # fp32 values; the reference widened them
    cfg = P.PcaConfig(k=8, oversample=6, block_size=7, seed=2)
    if source == "array":
        st = P.ArrayRowStream(a)
    elif source == "device":
        st = P.DeviceRowStream(torch.from_numpy(a).cuda())
    elif source == "generator":
        st = P.GeneratorRowStream(iter([a[:150], a[150:]]), n_cols=a.shape[1])
    else:
        p = tmp_path / "a.spca"
        P.matfile.write_matrix(p, a, dtype="float64")
        st = P.FileRowStream(p, buffer_bytes=100 * a.shape[1] * 8)
    res = P.single_pass_pca(P.NormalizedRowStream(st), cfg, block_rows=64)
    assert rel(res.s, golden_f["ns_s"]) <= 1e-10
    assert O.subspace_angle(res.u, golden_f["ns_u"]) <= 1e-10
    assert O.subspace_angle(res.v, golden_f["ns_v"]) <= 1e-10


@pytest.mark.parametrize("precision", PRECISIONS_F32)
def test_normalized_stream_fp32_file(golden_f, tmp_path, precision):
    if precision == "tc" and not _tc_ok():
        pytest.skip("no tensor-core path")
    a = golden_f["ns_a"]
    p = tmp_path / "a32.spca"
    P.matfile.write_matrix(p, a, dtype="float32")
    cfg = P.PcaConfig(k=8, oversample=6, block_size=7, seed=2)
    res = P.single_pass_pca(P.NormalizedRowStream(P.FileRowStream(p)), cfg, precision=precision)
    assert rel(res.s, golden_f["ns32_s"]) <= 1e-4
    assert O.subspace_angle(res.u, golden_f["ns32_u"]) <= 1e-4
    assert O.subspace_angle(res.v, golden_f["ns32_v"]) <= 1e-4


@pytest.mark.parametrize("tag,kw", [("c", {}), ("n", {"normalize": True}), ("p", {"power": 1}),
                                    ("nc", {"center": False})])
def test_estimator_matches_reference(golden_f, tag, kw):
    from sklearn.base import clone
    a = golden_f["ns_a"]
    est = P.SinglePassPCA(n_components=8, oversample=6, block_size=7, seed=3, **kw)
    est = clone(est).fit(a.astype(np.float64))
    assert rel(est.singular_values_, golden_f[f"est_{tag}_sv"]) <= 1e-10
    assert rel(est.explained_variance_, golden_f[f"est_{tag}_ev"]) <= 1e-10
    assert np.allclose(est.mean_, golden_f[f"est_{tag}_mean"], rtol=1e-12, atol=1e-15)
    assert O.subspace_angle(est.components_.T, golden_f[f"est_{tag}_components"].T) <= 1e-10
    assert np.allclose(est.components_, golden_f[f"est_{tag}_components"], atol=1e-9)  # signs too
    assert list(golden_f[f"est_{tag}_meta"]) == [est.n_samples_, est.n_passes_, est.retained_floats_]
    assert np.allclose(est.transform(golden_f["est_x2"]), golden_f[f"est_{tag}_t"], rtol=1e-9, atol=1e-11)
    assert np.allclose(est.inverse_transform(golden_f["est_z"]), golden_f[f"est_{tag}_it"], rtol=1e-9,
                       atol=1e-11)


def test_estimator_errors():
    est = P.SinglePassPCA(n_components=2)
    with pytest.raises(P.DimensionError):
        est.fit(np.ones(5))
    with pytest.raises(P.DataError):
        est.fit(np.array([[1.0, np.nan], [0.0, 1.0]]))
    from sklearn.exceptions import NotFittedError
    with pytest.raises(NotFittedError):
        est.transform(np.ones((2, 2)))
    est.fit(O.gaussian(30, 24, seed=5))
    with pytest.raises(P.DimensionError):
        est.transform(np.ones((2, 5)))


@pytest.mark.parametrize("l", [16, 200])
def test_tc_wide_n(l):
    """n wide enough that ~32-block K segments would outnumber the CTA pairs:
    the schedule lengthens the segments (S <= pairs / 2) instead of letting a
    G epilogue wait on its own pair's later unit."""
    if not _tc_ok():
        pytest.skip("no tensor-core path")
    m, n = 600, 80000
    a = O.gaussian(m, n, seed=41).astype(np.float32)
    om = O.gaussian(n, l, seed=42)
    st = P.sketch_pass(P.ArrayRowStream(a), om, precision="tc")
    ref = O.oracle_sketch(O.row_blocks(a, 4096), om.astype(np.float32).astype(np.float64))
    assert rel(st.g, ref.g) <= 2e-5 and rel(st.h, ref.h) <= 2e-5


@pytest.mark.parametrize("precision", ["tc", "simt"])
@pytest.mark.parametrize("m,n,l", [(5000, 1000, 60), (3000, 4096, 120), (2100, 2000, 250), (1000, 96, 16)])
def test_fused_normalisation_vs_oracle(precision, m, n, l):
    """spca_sketch_set_normalize: the sketch of normalize_rows(A) — fused into
    the pass kernel on the tensor-core path — against the oracle sketch of the
    explicitly normalized rows; rows with offsets, constant and zero rows."""
    if precision == "tc" and not _tc_ok():
        pytest.skip("no tensor-core path")
    rng = np.random.default_rng(m + n)
    a = (O.gaussian(m, n, seed=m) * rng.uniform(0.1, 10, size=(m, 1)) + rng.normal(0, 30, size=(m, 1)))
    a = a.astype(np.float32)
    a[7] = 2.5
    a[11] = 0.0
    om = O.gaussian(n, l, seed=n)
    st = P.sketch_pass(P.NormalizedRowStream(P.ArrayRowStream(a)), om, precision=precision)
    ref = O.oracle_sketch(O.row_blocks(O.oracle_normalize_rows(a.astype(np.float64)), 4096),
                          om.astype(np.float32).astype(np.float64))
    tol = 2e-5
    assert rel(st.g, ref.g) <= tol, rel(st.g, ref.g)
    assert rel(st.h, ref.h) <= tol, rel(st.h, ref.h)
    assert np.abs(st.col_sums - ref.col_sums).max() <= 1e-5 * np.sqrt(m), np.abs(st.col_sums - ref.col_sums).max()
    assert not np.asarray(st.g)[7].any() and not np.asarray(st.g)[11].any()


def test_fused_normalisation_bitwise_and_sources(tmp_path):
    """Same rows from host, device, pinned and file sources and any push
    split: bitwise identical normalized sketches; repeatable run to run."""
    if not _tc_ok():
        pytest.skip("no tensor-core path")
    a = (O.gaussian(9000, 700, seed=5) + 3.0).astype(np.float32)
    om = O.gaussian(700, 40, seed=6)
    base = P.sketch_pass(P.NormalizedRowStream(P.ArrayRowStream(a)), om)
    p = tmp_path / "a.spca"
    P.matfile.write_matrix(p, a, dtype="float32")
    for src in (P.DeviceRowStream(torch.from_numpy(a).cuda()), P.PinnedRowStream(torch.from_numpy(a)),
                P.FileRowStream(p, buffer_bytes=777 * 700 * 4),
                P.GeneratorRowStream(iter([a[:1234], a[1234:5000], a[5000:]]), n_cols=700, dtype=np.float32)):
        st = P.sketch_pass(P.NormalizedRowStream(src), om)
        for x, y in ((st.g, base.g), (st.h, base.h), (st.col_sums, base.col_sums)):
            assert np.array_equal(x, y)
    again = P.sketch_pass(P.NormalizedRowStream(P.ArrayRowStream(a)), om)
    assert np.array_equal(again.h, base.h)


# ----------------------------------------------------------- edge cases (f)
def test_empty_file_and_counters(tmp_path):
    p = tmp_path / "empty.spca"
    P.matfile.write_matrix(p, np.zeros((0, 8)), dtype="float32")
    st = P.sketch_pass(P.FileRowStream(p), O.gaussian(8, 4, seed=1))
    assert st.rows_seen == 0 and np.asarray(st.g).shape == (0, 4)
    with pytest.raises(P.EmptyStreamError):
        P.single_pass_pca(P.FileRowStream(p), P.PcaConfig(k=2, oversample=1, block_size=1))
    # pass counters around a normalized stream, both nestings
    a = O.gaussian(300, 40, seed=2).astype(np.float32)
    om = O.gaussian(40, 8, seed=3)
    outer = P.PassCounter(P.NormalizedRowStream(P.ArrayRowStream(a)))
    inner = P.PassCounter(P.ArrayRowStream(a))
    s1 = P.sketch_pass(outer, om)
    s2 = P.sketch_pass(P.NormalizedRowStream(inner), om)
    assert outer.passes_completed == 1 and outer.rows_read == 300
    assert inner.passes_completed == 1 and inner.rows_read == 300
    assert np.array_equal(s1.h, s2.h)


def test_normalize_single_column_and_state_errors():
    # one column: every row is constant -> the zero row (SIMT: n not a multiple of 4)
    a = O.gaussian(50, 1, seed=4)
    st = P.sketch_pass(P.NormalizedRowStream(P.ArrayRowStream(a)), O.gaussian(1, 1, seed=5))
    assert not np.asarray(st.g).any() and not np.asarray(st.h).any()
    sk = P.GpuSketch(16, O.gaussian(16, 4, seed=6), np.float32)
    sk.push(np.ones((3, 16), np.float32), 0)
    with pytest.raises(P.DeviceError):
        _lib_set_normalize(sk)
    sk.close()


def _lib_set_normalize(sk):
    from paper_1704_07669_b200 import _lib
    _lib.check(sk.lib.spca_sketch_set_normalize(sk.h, 1), sk.h)


def test_power_refine_normalized_file(tmp_path):
    """Two passes over a normalized file stream: the same factorisation as
    power_refine over the explicitly normalized rows in memory."""
    rng = np.random.default_rng(7)
    a = (rng.standard_normal((900, 60)) @ np.diag(1.0 / np.arange(1, 61)) @ rng.standard_normal((60, 256))
         + rng.normal(0, 2, size=(900, 1))).astype(np.float32)
    p = tmp_path / "a.spca"
    P.matfile.write_matrix(p, a, dtype="float32")
    cfg = P.PcaConfig(k=8, oversample=8, block_size=8, power=1, seed=4)
    pc = P.PassCounter(P.FileRowStream(p))
    res = P.power_refine(P.NormalizedRowStream(pc), cfg)
    want = P.power_refine(O.oracle_normalize_rows(a.astype(np.float64)).astype(np.float32), cfg)
    assert pc.passes_completed == 2
    assert rel(res.s, want.s) <= 1e-4
    assert O.subspace_angle(res.v, want.v) <= 1e-3


# ------------------------------------------- full-size properties (cfg3, cfg5)
@pytest.mark.gpu
@pytest.mark.parametrize("config", ["cfg3", "cfg5"])
def test_full_size_properties(config):
    """BASELINE configs 3 (1 000 000 x 4096, l = 120) and 5 (50 000 x 200 000,
    l = 250, column groups) at full size on one device, through
    size-independent identities in fp64: G = A Omega and y^T H x = (A y)^T (G x)
    on random probes, Omega^T H = G^T G (both equal Omega^T A^T A Omega), column
    sums against a direct reduction, bitwise repeatability."""
    if not _tc_ok():
        pytest.skip("no tensor-core path")
    from paper_1704_07669_b200 import synth
    cs = synth.config_shape(config)
    a = synth.config_matrix(config, device="cuda")
    m, n = a.shape
    l = cs["l"]
    om = O.gaussian(n, l, 1)
    st = P.sketch_pass(P.DeviceRowStream(a), om, keep_on_device=True)
    om32 = st.omega
    gen = torch.Generator(device="cuda").manual_seed(0)
    x = torch.randn(l, 4, device="cuda", dtype=torch.float64, generator=gen)
    y = torch.randn(n, 4, device="cuda", dtype=torch.float64, generator=gen)
    step = max(1, int(2e8) // n)
    rows = min(m, 20 * step)
    g_ref = a[:rows].double() @ (om32 @ x)
    assert float(torch.linalg.norm(st.g[:rows] @ x - g_ref) / torch.linalg.norm(g_ref)) < 2e-5
    ay = torch.cat([a[i:i + step].double() @ y for i in range(0, m, step)])
    rhs = ay.T @ (st.g @ x)
    assert float(torch.linalg.norm(y.T @ st.h @ x - rhs) / torch.linalg.norm(rhs)) < 1e-5
    cross, gram = om32.T @ st.h, st.g.T @ st.g
    assert float(torch.linalg.norm(cross - gram) / torch.linalg.norm(gram)) < 1e-5
    cs_ref = torch.zeros(n, dtype=torch.float64, device="cuda")
    for i in range(0, m, step):
        cs_ref += a[i:i + step].double().sum(dim=0)
    assert float(torch.linalg.norm(st.col_sums - cs_ref) / torch.linalg.norm(cs_ref)) < 1e-6
    st2 = P.sketch_pass(P.DeviceRowStream(a), om, keep_on_device=True)
    assert torch.equal(st.h, st2.h) and torch.equal(st.g, st2.g) and torch.equal(st.col_sums, st2.col_sums)
    del a, st, st2, ay
    torch.cuda.empty_cache()


def test_merged_column_groups_bitwise_equal_to_one_launch_per_group(tmp_path):
    """l > 128 (column groups of 128): the merged launch (every group in one
    pass-kernel launch, csrc/tc_host.cuh tc_merged_groups) gives the same
    G, H and column sums bit for bit as one launch per group
    (SPCA_TC_SEQ_GROUPS=1, read once per process: a subprocess each)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    script = r'''
import sys, numpy as np, torch
sys.path.insert(0, %r)
import paper_1704_07669_b200 as P
m, n, l = 3000, 2000, 300
gen = torch.Generator(device="cuda").manual_seed(4)
a = torch.randn(m, n, device="cuda", dtype=torch.float32, generator=gen)
om = np.random.default_rng(5).standard_normal((n, l))
sk = P.GpuSketch(n, om, np.float32, precision="tc", rows_hint=m)
sk.push(a, 0, final=True)
g, h, cs, rows = sk.finish(on_device=True)
np.savez(sys.argv[1], g=g.cpu().numpy(), h=h.cpu().numpy(), cs=cs.cpu().numpy())
''' % root
    outs = []
    for seq in (False, True):
        env = dict(os.environ)
        env.pop("SPCA_TC_SEQ_GROUPS", None)
        if seq:
            env["SPCA_TC_SEQ_GROUPS"] = "1"
        out = str(tmp_path / f"sk_{int(seq)}.npz")
        subprocess.run([sys.executable, "-c", script, out], env=env, check=True, timeout=300)
        outs.append(np.load(out))
    for k in ("g", "h", "cs"):
        assert np.array_equal(outs[0][k], outs[1][k]), k
