"""Matrix-file formats and FileRowStream (host side; no GPU).

Pinned against files written by the reference's own writers
(tests/golden/make_matfile_golden.py) and restating the reference's
tests/test_streams.py matfile / FileRowStream cases."""
import os

import numpy as np
import pytest

from paper_1704_07669_b200 import FileRowStream, FormatError, StreamFormatError, matfile

GOLD = os.path.join(os.path.dirname(__file__), "golden", "matfile")


@pytest.fixture(scope="module")
def inputs():
    return np.load(os.path.join(GOLD, "inputs.npz"))


def _collect(stream, br):
    return np.vstack([b.values for b in stream.blocks(br)])


class TestGolden:
    def test_reads_reference_files(self, inputs):
        lay = matfile.read_header(os.path.join(GOLD, "ref_f64.spca"))
        assert (lay.rows, lay.cols, lay.dtype, lay.offset) == (7, 5, np.dtype("<f8"), 22)
        assert np.array_equal(matfile.read_matrix(os.path.join(GOLD, "ref_f64.spca")), inputs["a64"])
        want32 = inputs["a32"].astype(np.float32).astype(np.float64)
        assert np.array_equal(matfile.read_matrix(os.path.join(GOLD, "ref_f32.spca")), want32)
        raw = matfile.read_matrix(os.path.join(GOLD, "ref_f32.raw"), rows=6, cols=4, dtype="float32")
        assert np.array_equal(raw, want32)

    @pytest.mark.parametrize("name,key,dtype,header", [
        ("ref_f64.spca", "a64", "float64", True),
        ("ref_f32.spca", "a32", "float32", True),
        ("ref_f32.raw", "a32", "float32", False),
    ])
    def test_writer_bytes_identical(self, tmp_path, inputs, name, key, dtype, header):
        p = tmp_path / name
        matfile.write_matrix(p, inputs[key], dtype=dtype, header=header)
        with open(os.path.join(GOLD, name), "rb") as fh:
            assert p.read_bytes() == fh.read()

    def test_sigma_csv(self, tmp_path, inputs):
        p = tmp_path / "s.csv"
        matfile.write_sigma_csv(p, inputs["sig"])
        with open(os.path.join(GOLD, "sigma.csv"), "rb") as fh:
            assert p.read_bytes() == fh.read()
        assert np.array_equal(matfile.read_sigma_csv(os.path.join(GOLD, "sigma.csv")), inputs["sig"])


class TestMatfile:  # the reference's test_streams.py TestMatfile cases
    def test_header_roundtrip(self, tmp_path):
        a = np.random.default_rng(1).standard_normal((7, 5))
        p = tmp_path / "m.spca"
        matfile.write_matrix(p, a, dtype="float64", header=True)
        lay = matfile.read_header(p)
        assert (lay.rows, lay.cols, lay.offset) == (7, 5, matfile.HEADER_BYTES)
        assert np.array_equal(matfile.read_matrix(p), a)

    def test_known_bytes(self, tmp_path):
        p = tmp_path / "fixed.bin"
        vals = np.arange(12, dtype="<f4").reshape(4, 3)
        p.write_bytes(vals.tobytes())
        back = matfile.read_matrix(p, rows=4, cols=3, dtype="float32")
        assert back.dtype == np.float64 and np.array_equal(back, vals.astype(np.float64))

    def test_size_mismatch(self, tmp_path):
        p = tmp_path / "bad.bin"
        p.write_bytes(b"\x00" * 10)
        with pytest.raises(FormatError):
            matfile.raw_layout(p, rows=4, cols=3, dtype="float32")

    @pytest.mark.parametrize("blob", [
        b"NOPE" + b"\x00" * 30,                               # magic
        b"SPCA\x02" + b"\x00" * 17,                           # version
        b"SPCA\x01" + (1).to_bytes(8, "little") * 2 + b"\x03",  # dtype code
        b"SPCA\x01" + (2).to_bytes(8, "little") * 2 + b"\x08",  # size
        b"SPCA",                                              # too short
    ])
    def test_bad_headers(self, tmp_path, blob):
        p = tmp_path / "bad.spca"
        p.write_bytes(blob)
        with pytest.raises(FormatError):
            matfile.read_header(p)

    def test_sniff(self, tmp_path):
        a = np.random.default_rng(3).standard_normal((6, 2))
        p = tmp_path / "m.bin"
        matfile.write_matrix(p, a, dtype="float64", header=False)
        assert matfile.sniff_layout(p, rows=6, cols=2, dtype="float64").offset == 0
        q = tmp_path / "z.bin"
        q.write_bytes(b"\x00" * 16)
        with pytest.raises(FormatError):
            matfile.sniff_layout(q)

    def test_bad_dtype_and_dims(self, tmp_path):
        p = tmp_path / "m.bin"
        p.write_bytes(b"\x00" * 16)
        with pytest.raises(FormatError):
            matfile.raw_layout(p, rows=2, cols=2, dtype="int32")
        with pytest.raises(FormatError):
            matfile.raw_layout(p, rows=0, cols=2, dtype="float32")

    def test_sigma_csv_errors(self, tmp_path):
        p = tmp_path / "s.csv"
        p.write_text("1,2.0\n3,1.0\n")
        with pytest.raises(FormatError):
            matfile.read_sigma_csv(p)
        p.write_text("1;2.0\n")
        with pytest.raises(FormatError):
            matfile.read_sigma_csv(p)


class TestFileRowStream:
    def test_matches_memory_matrix(self, tmp_path):
        a = np.random.default_rng(4).standard_normal((10, 6))
        p = tmp_path / "a.spca"
        matfile.write_matrix(p, a, dtype="float64")
        s = FileRowStream(p)
        assert (s.n_rows, s.n_cols, s.resettable, s.dtype) == (10, 6, True, np.float64)
        for br in (1, 4, 10, 11):
            assert np.array_equal(_collect(s, br), a)
        assert s.bytes_read == 4 * 10 * 6 * 8 and s.read_seconds >= 0.0

    def test_float32_file(self, tmp_path):
        a = np.random.default_rng(5).standard_normal((40, 3))
        p = tmp_path / "a.bin"
        matfile.write_matrix(p, a, dtype="float32", header=False)
        s = FileRowStream(p, rows=40, cols=3, dtype="float32", read_threads=3)
        assert s.dtype == np.float32  # what the device pass computes in
        got = _collect(s, 7)
        assert got.dtype == np.float64  # blocks widen like the reference
        assert np.array_equal(got, a.astype(np.float32).astype(np.float64))

    def test_parallel_reads(self, tmp_path):
        a = np.random.default_rng(6).standard_normal((3000, 17)).astype(np.float32)
        p = tmp_path / "a.spca"
        matfile.write_matrix(p, a, dtype="float32")
        s = FileRowStream(p, read_threads=4)
        out = np.empty((2999, 17), np.float32)
        from concurrent.futures import ThreadPoolExecutor
        with ThreadPoolExecutor(4) as pool:
            s.read_rows_into(out, 1, 2999, pool)
        assert np.array_equal(out, a[1:])

    def test_truncated_after_open(self, tmp_path):
        a = np.ones((8, 4))
        p = tmp_path / "a.spca"
        matfile.write_matrix(p, a, dtype="float64")
        s = FileRowStream(p)
        with open(p, "r+b") as fh:
            fh.truncate(matfile.HEADER_BYTES + 8 * 4 * 5)
        with pytest.raises(FormatError):
            _collect(s, 3)

    def test_declared_size_mismatch(self, tmp_path):
        p = tmp_path / "a.bin"
        p.write_bytes(b"\x00" * 24)
        with pytest.raises(FormatError):
            FileRowStream(p, rows=5, cols=5, dtype="float64")

    def test_missing_file(self, tmp_path):
        with pytest.raises(OSError):
            FileRowStream(tmp_path / "absent.spca")

    def test_bad_block_rows(self, tmp_path):
        p = tmp_path / "a.spca"
        matfile.write_matrix(p, np.ones((2, 2)), dtype="float64")
        with pytest.raises(StreamFormatError):
            list(FileRowStream(p).blocks(0))
