"""CPU-side checks of the boundary: the C-ABI library loads and exports every
symbol include/spca.h declares, the Python mirror exposes the reference's
hot-path names with compatible signatures, and host logic behaves without a
GPU (no compute calls)."""

import inspect
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "spca.h")
LIB = os.path.join(ROOT, "paper_1704_07669_b200", "libspca.so")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(spca_[a-z_0-9]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    from paper_1704_07669_b200 import build
    build.build()
    from paper_1704_07669_b200 import _lib
    return _lib.load()


def test_header_symbols_exported(lib):
    syms = declared_symbols()
    assert len(syms) >= 14
    out = subprocess.run(["nm", "-D", "--defined-only", LIB], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (spca_\w+)", out))
    missing = [s for s in syms if s not in exported]
    assert not missing, missing
    from paper_1704_07669_b200 import _lib
    assert sorted(_lib.SIGNATURES) == syms


def test_abi_version_and_info(lib):
    assert lib.spca_abi_version() == 1
    assert b"sm_100a" in lib.spca_build_info()


def test_create_without_gpu_fails_cleanly(lib):
    """No device here: create must return a CUDA error code, not crash, and
    the Python layer must raise (there is no CPU fallback)."""
    from paper_1704_07669_b200 import _lib
    import ctypes
    h = ctypes.c_void_p()
    om = np.ones((4, 2))
    rc = lib.spca_sketch_create(ctypes.byref(h), 4, 2, 0, 1, om.ctypes.data_as(ctypes.c_void_p),
                                _lib.MEM_PAGEABLE, 0, None, 0, 0)
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:
        has_gpu = False
    if has_gpu:
        pytest.skip("GPU present")
    assert rc != 0 and not h.value
    code, row, msg = _lib.last_error(None)
    assert code == rc and msg


def test_argument_errors_map_to_reference_classes(lib):
    from paper_1704_07669_b200 import _lib
    from paper_1704_07669_b200.errors import ConfigError, StreamFormatError
    import ctypes
    h = ctypes.c_void_p()
    om = np.ones((4, 2))
    rc = lib.spca_sketch_create(ctypes.byref(h), 0, 2, 0, 1, om.ctypes.data_as(ctypes.c_void_p),
                                _lib.MEM_PAGEABLE, 0, None, 0, 0)
    with pytest.raises(StreamFormatError):
        _lib.check(rc)
    rc = lib.spca_sketch_create(ctypes.byref(h), 4, 2, 7, 1, om.ctypes.data_as(ctypes.c_void_p),
                                _lib.MEM_PAGEABLE, 0, None, 0, 0)
    with pytest.raises(ConfigError):
        _lib.check(rc)


def test_public_api_mirrors_reference_signatures():
    import paper_1704_07669_b200 as P
    for name in ("single_pass_pca", "sketch_pass", "PcaConfig", "TruncatedSvd", "SketchState",
                 "blocked_qb", "center_correct", "ArrayRowStream", "GeneratorRowStream",
                 "PassCounter", "RowBlock", "RowStream", "DataError", "StreamFormatError",
                 "EmptyStreamError", "ConfigError", "RankDeficiencyError", "CapabilityError"):
        assert hasattr(P, name), name
    sig = inspect.signature(P.single_pass_pca)
    assert list(sig.parameters)[:6] == ["data", "cfg", "block_rows", "fixed_order",
                                       "on_deficiency", "compensated"]
    assert sig.parameters["on_deficiency"].default == "repair"
    sig = inspect.signature(P.sketch_pass)
    assert list(sig.parameters)[:5] == ["stream", "omega", "block_rows", "fixed_order", "compensated"]


def test_pca_config_semantics():
    from paper_1704_07669_b200 import ConfigError, PcaConfig
    assert PcaConfig(k=20, oversample=10, block_size=10).l == 30
    assert PcaConfig(k=50, oversample=10).l == 60
    assert PcaConfig(k=100, oversample=20).l == 120
    assert PcaConfig(k=200, oversample=50).l == 250
    assert PcaConfig(k=7, oversample=4, block_size=5).l == 15
    for bad in (dict(k=0), dict(k=1, oversample=-1), dict(k=1, block_size=0), dict(k=1, power=2),
                dict(k=1, seed=-1)):
        with pytest.raises(ConfigError):
            PcaConfig(**bad)
    with pytest.raises(ConfigError):
        PcaConfig(k=45, oversample=10).validate_dims(50, 200)
    PcaConfig(k=40, oversample=10).validate_dims(50, 200)
    PcaConfig(k=40, oversample=10).validate_dims(50, None)


def test_streams_contract():
    from paper_1704_07669_b200 import (ArrayRowStream, CapabilityError, GeneratorRowStream,
                                       PassCounter, StreamFormatError)
    a = np.arange(30.0).reshape(10, 3)
    s = ArrayRowStream(a)
    blocks = list(s.blocks(4))
    assert [b.first_row_index for b in blocks] == [0, 4, 8]
    assert np.array_equal(np.vstack([b.values for b in blocks]), a)
    assert ArrayRowStream(a.astype(np.float32)).dtype == np.float32
    assert ArrayRowStream(a.astype(np.int64)).dtype == np.float64
    g = GeneratorRowStream(iter([a[:3], a[3:]]), n_cols=3)
    assert g.n_rows is None and not g.resettable
    pc = PassCounter(g)
    assert sum(b.values.shape[0] for b in pc.blocks(2)) == 10
    assert g.n_rows == 10 and pc.passes_completed == 1
    with pytest.raises(CapabilityError):
        list(g.blocks(2))
    with pytest.raises(StreamFormatError):
        list(GeneratorRowStream(iter([np.ones((2, 4))]), n_cols=3).blocks(2))
    with pytest.raises(StreamFormatError):
        ArrayRowStream(np.ones(5))
    pc2 = PassCounter(ArrayRowStream(a))
    kind, mat = pc2.whole()
    assert kind == "host" and pc2.passes_completed == 1 and pc2.rows_read == 10


def test_gaussian_matrix_is_reference_rng(golden):
    """Omega comes from the reference's own generator (bits pinned by the
    golden hashes of the reference run)."""
    import hashlib
    from paper_1704_07669_b200 import gaussian_matrix
    _, meta = golden
    om = gaussian_matrix(10000, 60, 1)
    assert hashlib.sha256(om.tobytes()).hexdigest()[:16] == meta["omega_cfg2_s1_f64"]


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_1704_07669_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith(".py"):
                src = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(from|import)\s+oracle\b", src, re.M), f


def test_basic_and_legacy_stream_contracts_before_the_device():
    """CapabilityError for a one-shot stream (basic_rand_svd, algorithms.py:218-219)
    and for an unknown row count (legacy_single_pass, :326-331) — raised before
    any device work, as the reference does."""
    import numpy as np
    import paper_1704_07669_b200 as P

    def gen():
        yield np.zeros((3, 4))
    cfg = P.PcaConfig(k=1, oversample=1, block_size=1)
    one_shot = P.GeneratorRowStream(gen(), n_cols=4)
    with pytest.raises(P.CapabilityError, match="resettable"):
        P.basic_rand_svd(one_shot, cfg)
    with pytest.raises(P.CapabilityError, match="row count up front"):
        P.legacy_single_pass(P.GeneratorRowStream(gen(), n_cols=4), cfg)
