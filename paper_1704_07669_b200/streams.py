"""Row-block streams — the input boundary of the sketch pass.

Mirrors the ``RowStream`` protocol of the reference
(/root/reference/pkg/src/streampca/streams.py:23-221): consecutive,
non-overlapping ``RowBlock``s covering the matrix top to bottom; ``n_rows``
may be ``None`` until a one-shot source is exhausted; ``PassCounter`` counts
completed traversals.

Differences, all additive:
  * streams carry a ``dtype`` (float32 or float64). The reference widens
    every block to float64 (streams.py:59,128); here float32 data stays
    float32 and takes the fp32 device path (BASELINE configs 2-5).
  * ``DeviceRowStream`` (rows already in HBM) and ``PinnedRowStream`` (rows
    in page-locked host memory, streamed over PCIe) feed the GPU directly.
  * ``FileRowStream`` keeps the file's element type and also offers
    ``read_rows_into`` (parallel positional reads into a caller's buffer),
    which the pass uses to fill pinned buffers without a host-side copy.
  * in-memory streams expose ``whole()`` so a pass can hand the library the
    full matrix in one push; the library re-chunks canonically, so results
    are bitwise identical to a block-by-block traversal.
Any object with ``n_rows``, ``n_cols``, ``resettable`` and ``blocks()``
(including the reference's own stream classes) is accepted by sketch_pass.
"""

from __future__ import annotations

import os
import time
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass
from typing import Any, Iterator, Optional

import numpy as np

from . import matfile
from .errors import CapabilityError, FormatError, StreamFormatError


@dataclass(frozen=True)
class RowBlock:
    """Rows first_row_index .. first_row_index + len(values) - 1 (streams.py:23-28).
    ``values`` is a 2-d numpy array or torch tensor."""

    first_row_index: int
    values: Any


class RowStream:
    """Source of row blocks (streams.py:31-52)."""

    @property
    def n_rows(self) -> Optional[int]:
        raise NotImplementedError

    @property
    def n_cols(self) -> int:
        raise NotImplementedError

    @property
    def resettable(self) -> bool:
        raise NotImplementedError

    @property
    def dtype(self) -> np.dtype:
        return np.dtype(np.float64)

    def blocks(self, block_rows: int) -> Iterator[RowBlock]:
        raise NotImplementedError


def _float_dtype(dt) -> np.dtype:
    dt = np.dtype(dt)
    return dt if dt in (np.dtype(np.float32), np.dtype(np.float64)) else np.dtype(np.float64)


class ArrayRowStream(RowStream):
    """Resettable stream over an in-memory host matrix (streams.py:55-80).
    float32 input stays float32; everything else becomes float64."""

    def __init__(self, a):
        a = np.asarray(a)
        a = np.asarray(a, dtype=_float_dtype(a.dtype))
        if a.ndim != 2 or a.shape[1] < 1:
            raise StreamFormatError("ArrayRowStream expects a 2-d matrix with columns")
        if a.strides[1] != a.itemsize or a.strides[0] < a.shape[1] * a.itemsize:
            a = np.ascontiguousarray(a)
        self._a = a
        self.whole_passes = 0

    @property
    def n_rows(self) -> int:
        return self._a.shape[0]

    @property
    def n_cols(self) -> int:
        return self._a.shape[1]

    @property
    def resettable(self) -> bool:
        return True

    @property
    def dtype(self) -> np.dtype:
        return self._a.dtype

    def blocks(self, block_rows: int) -> Iterator[RowBlock]:
        if block_rows < 1:
            raise StreamFormatError("block_rows must be >= 1")
        for start in range(0, self._a.shape[0], block_rows):
            yield RowBlock(start, self._a[start:start + block_rows])

    def whole(self):
        """("host", matrix) — one full pass handed over at once."""
        self.whole_passes += 1
        return "host", self._a


class _TorchRowStream(RowStream):
    _kind = "device"

    def __init__(self, t):
        import torch
        if not isinstance(t, torch.Tensor) or t.dim() != 2 or t.shape[1] < 1:
            raise StreamFormatError(f"{type(self).__name__} expects a 2-d torch tensor")
        if t.dtype not in (torch.float32, torch.float64):
            raise StreamFormatError("rows must be float32 or float64")
        if t.stride(1) != 1:
            t = t.contiguous()
        self._t = t
        self.whole_passes = 0

    @property
    def n_rows(self) -> int:
        return int(self._t.shape[0])

    @property
    def n_cols(self) -> int:
        return int(self._t.shape[1])

    @property
    def resettable(self) -> bool:
        return True

    @property
    def dtype(self) -> np.dtype:
        import torch
        return np.dtype(np.float32 if self._t.dtype == torch.float32 else np.float64)

    @property
    def tensor(self):
        return self._t

    def blocks(self, block_rows: int) -> Iterator[RowBlock]:
        if block_rows < 1:
            raise StreamFormatError("block_rows must be >= 1")
        for start in range(0, self.n_rows, block_rows):
            yield RowBlock(start, self._t[start:start + block_rows])

    def whole(self):
        self.whole_passes += 1
        return self._kind, self._t


class DeviceRowStream(_TorchRowStream):
    """Rows resident in GPU memory (a CUDA torch tensor, row-major)."""

    _kind = "device"

    def __init__(self, t):
        super().__init__(t)
        if not self._t.is_cuda:
            raise StreamFormatError("DeviceRowStream needs a CUDA tensor")


class PinnedRowStream(_TorchRowStream):
    """Rows in page-locked host memory; the pass streams them over PCIe with
    double-buffered asynchronous copies (the out-of-HBM mode, config 4)."""

    _kind = "pinned"

    def __init__(self, t):
        super().__init__(t)
        if self._t.is_cuda:
            raise StreamFormatError("PinnedRowStream needs a host tensor")
        if not self._t.is_pinned():
            self._t = self._t.pin_memory()


class FileRowStream(RowStream):
    """Rows of a matrix file, raw or self-describing (streams.py:83-128,
    layouts in matfile.py). Resettable. ``read_seconds`` / ``bytes_read``
    account the time spent in file reads, as in the reference.

    ``blocks`` widens to float64 exactly as the reference does (:128). The
    device pass does not use it: it calls ``read_rows_into`` to fill
    page-locked buffers in the file's own element type (``dtype``: float32
    files are sketched in fp32, like every other float32 source), with no
    widening and no host-side copy (sketch.py ``_push_file``)."""

    def __init__(self, path, rows=None, cols=None, dtype=None, layout=None, read_threads: Optional[int] = None,
                 buffer_bytes: int = 64 << 20):
        self._path = str(path)
        self.buffer_bytes = max(1, int(buffer_bytes))  # page-locked buffer size of the device pass
        self._layout = layout if layout is not None else matfile.sniff_layout(self._path, rows, cols, dtype)
        self.read_seconds = 0.0
        self.bytes_read = 0
        # parallel positional reads from the page cache: 16 threads 35.9 GB/s,
        # 8 31.1, 4 23.7 at config 2 (tools/file_bench.py, 16-core host)
        if read_threads is None:
            read_threads = min(16, os.cpu_count() or 1)
        self.read_threads = max(1, int(read_threads))

    @property
    def layout(self) -> matfile.FileLayout:
        return self._layout

    @property
    def path(self) -> str:
        return self._path

    @property
    def n_rows(self) -> int:
        return self._layout.rows

    @property
    def n_cols(self) -> int:
        return self._layout.cols

    @property
    def resettable(self) -> bool:
        return True

    @property
    def dtype(self) -> np.dtype:
        return np.dtype(self._layout.dtype.newbyteorder("="))

    def read_rows_into(self, out: np.ndarray, start: int, rows: int, pool=None) -> None:
        """Read rows [start, start + rows) into the C-contiguous ``out``
        (at least rows x n_cols of the file's dtype) with positional reads,
        split across ``pool`` threads when given. FormatError when the file
        ends early."""
        lay = self._layout
        nbytes = rows * lay.row_bytes
        dst = memoryview(out.reshape(-1).view(np.uint8))[:nbytes]
        base = lay.offset + start * lay.row_bytes
        t0 = time.perf_counter()
        fd = os.open(self._path, os.O_RDONLY)
        try:
            def span(lo, hi):
                pos = lo
                while pos < hi:
                    got = os.preadv(fd, [dst[pos:hi]], base + pos)
                    if got <= 0:
                        raise FormatError(f"{self._path}: truncated at row {start + pos // lay.row_bytes}")
                    pos += got
            parts = self.read_threads if pool is not None else 1
            step = -(-nbytes // parts)
            step = -(-step // 4096) * 4096  # page-aligned pieces
            cuts = [(lo, min(nbytes, lo + step)) for lo in range(0, nbytes, step)] or [(0, 0)]
            if pool is None or len(cuts) == 1:
                for lo, hi in cuts:
                    span(lo, hi)
            else:
                for f in [pool.submit(span, lo, hi) for lo, hi in cuts]:
                    f.result()
        finally:
            os.close(fd)
        self.read_seconds += time.perf_counter() - t0
        self.bytes_read += nbytes

    def blocks(self, block_rows: int) -> Iterator[RowBlock]:
        if block_rows < 1:
            raise StreamFormatError("block_rows must be >= 1")
        lay = self._layout
        with ThreadPoolExecutor(self.read_threads) as pool:
            for start in range(0, lay.rows, block_rows):
                rows = min(block_rows, lay.rows - start)
                buf = np.empty((rows, lay.cols), dtype=self.dtype)
                self.read_rows_into(buf, start, rows, pool)
                yield RowBlock(start, buf.astype(np.float64, copy=False))


class GeneratorRowStream(RowStream):
    """One-shot stream over an iterable of 2-d arrays (streams.py:140-181):
    not resettable; ``n_rows`` is known only after exhaustion."""

    def __init__(self, iterable, n_cols: int, dtype=np.float64):
        self._it = iter(iterable)
        self._n_cols = int(n_cols)
        self._n_rows: Optional[int] = None
        self._consumed = False
        self._dtype = _float_dtype(dtype)

    @property
    def n_rows(self) -> Optional[int]:
        return self._n_rows

    @property
    def n_cols(self) -> int:
        return self._n_cols

    @property
    def resettable(self) -> bool:
        return False

    @property
    def dtype(self) -> np.dtype:
        return self._dtype

    def blocks(self, block_rows: int) -> Iterator[RowBlock]:
        if self._consumed:
            raise CapabilityError("this stream supports a single pass only")
        self._consumed = True
        seen = 0
        for chunk in self._it:
            vals = np.asarray(chunk, dtype=self._dtype)
            if vals.ndim != 2 or vals.shape[1] != self._n_cols:
                raise StreamFormatError(
                    f"generator yielded shape {vals.shape}, expected (*, {self._n_cols})")
            for start in range(0, vals.shape[0], block_rows):
                part = vals[start:start + block_rows]
                yield RowBlock(seen, part)
                seen += part.shape[0]
        self._n_rows = seen


class PassCounter(RowStream):
    """Counts completed traversals and rows read (streams.py:184-221); a
    whole-matrix hand-over counts as one complete pass."""

    def __init__(self, wrapped):
        self.wrapped = wrapped
        self.passes_completed = 0
        self.rows_read = 0
        self.pass_in_progress = False

    @property
    def n_rows(self) -> Optional[int]:
        return self.wrapped.n_rows

    @property
    def n_cols(self) -> int:
        return self.wrapped.n_cols

    @property
    def resettable(self) -> bool:
        return self.wrapped.resettable

    @property
    def dtype(self) -> np.dtype:
        return getattr(self.wrapped, "dtype", np.dtype(np.float64))

    def blocks(self, block_rows: int) -> Iterator[RowBlock]:
        self.pass_in_progress = True
        rows_this_pass = 0
        for block in self.wrapped.blocks(block_rows):
            rows_this_pass += block.values.shape[0]
            self.rows_read += block.values.shape[0]
            yield block
        total = self.wrapped.n_rows
        if total is None or rows_this_pass == total:
            self.passes_completed += 1
            self.pass_in_progress = False

    def whole(self):
        if not hasattr(self.wrapped, "whole"):
            raise AttributeError("whole")
        kind, mat = self.wrapped.whole()
        self.rows_read += int(mat.shape[0])
        self.passes_completed += 1
        self.pass_in_progress = False
        return kind, mat


def has_whole(stream) -> bool:
    if isinstance(stream, PassCounter):
        return has_whole(stream.wrapped)
    return hasattr(stream, "whole")
