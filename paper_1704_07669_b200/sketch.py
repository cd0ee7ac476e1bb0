"""The one-pass sketch on the GPU — the drop-in for the reference's
``sketch_pass`` (/root/reference/pkg/src/streampca/sketch.py:52-116).

One traversal of the row stream accumulates, per row block A_i,

    G_i = A_i Omega,   H += A_i^T G_i,   col_sums += 1^T A_i

on one B200 through libspca.so (include/spca.h). Blocks are pushed as they
arrive; in-memory, device and pinned sources are handed over whole and the
library streams them in canonical chunks (pinned host rows go through
double-buffered async copies). Shape errors raise ``StreamFormatError`` and
the first non-finite row raises ``DataError(row=...)`` exactly as
``_check_block`` (sketch.py:40-49) does.

Precision: float64 data runs the fp64 DFMA path; float32 data runs the fp32
path (tensor cores with split precision when available, else FFMA), with
Omega rounded once to float32 — ``SketchState.omega`` records the Omega the
sketch actually used so the post-pass stays consistent with it.
"""

from __future__ import annotations

import ctypes
import queue
import threading
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, replace
from typing import Optional

import numpy as np

from . import _lib
from .device import default_device, host_copy, is_torch, to_device64, torch_mod
from .errors import EmptyStreamError, StreamFormatError
from .streams import FileRowStream, PassCounter, RowBlock, RowStream, has_whole

_PRECISIONS = {"auto": _lib.PREC_AUTO, "simt": _lib.PREC_SIMT, "tc": _lib.PREC_TC}


@dataclass(frozen=True)
class SketchState:
    """Accumulators after one pass (sketch.py:25-37). Arrays are numpy
    float64 by default, CUDA float64 tensors with ``keep_on_device``.
    ``omega`` (extra) is the test matrix exactly as the sketch used it."""

    g: object
    h: object
    col_sums: object
    rows_seen: int
    omega: object = None

    @property
    def retained_floats(self) -> int:
        """Floats held by the sketch itself, excluding Omega (sketch.py:34-37)."""
        size = (lambda a: int(a.numel()) if is_torch(a) else int(np.asarray(a).size))
        return size(self.g) + size(self.h) + size(self.col_sums)


class GpuSketch:
    """Owner of one libspca handle (single consumer, one GPU)."""

    def __init__(self, n: int, omega: np.ndarray, dtype, precision: str = "auto",
                 device=None, rows_hint: int = 0, compensated: bool = False, stream=None,
                 normalize: bool = False, shift: bool = False):
        torch = torch_mod()
        self.lib = _lib.load()
        self.device = default_device(device)
        self.n = int(n)
        om_dev = is_torch(omega) and omega.is_cuda  # drawn on the device (gaussian_matrix_device)
        if om_dev:
            om = omega.to(device=self.device, dtype=torch.float64).contiguous()
            om_ptr, om_where = ctypes.c_void_p(om.data_ptr()), _lib.MEM_DEVICE
        else:
            om = np.ascontiguousarray(np.asarray(omega, dtype=np.float64))
            om_ptr, om_where = om.ctypes.data_as(ctypes.c_void_p), _lib.MEM_PAGEABLE
        self.l = int(om.shape[1])
        self.dtype = np.dtype(dtype)
        if self.dtype not in (np.dtype(np.float32), np.dtype(np.float64)):
            raise StreamFormatError(f"unsupported element type {self.dtype}")
        code = _lib.SPCA_F32 if self.dtype == np.float32 else _lib.SPCA_F64
        prec = _PRECISIONS[precision] if isinstance(precision, str) else int(precision)
        if stream is None:
            stream = torch.cuda.current_stream(self.device)
        self.stream = stream
        handle = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            rc = self.lib.spca_sketch_create(
                ctypes.byref(handle), self.n, self.l, code, prec,
                om_ptr, om_where,
                # torch's default stream is the legacy NULL stream: hand the library
                # cudaStreamLegacy (0x1) so both order on it (NULL would mean a
                # private stream that does not synchronize with torch's work)
                self.device.index, ctypes.c_void_p(stream.cuda_stream or 1), int(rows_hint),
                1 if compensated else 0)
        _lib.check(rc)
        self.h = handle
        if normalize:  # rows are sketched as normalize_rows leaves them (fused on the TC path)
            _lib.check(self.lib.spca_sketch_set_normalize(self.h, 1), self.h)
        elif shift:  # accumulate A - 1 c^T (c = mean of the first rows), undone in fp64 at finish
            self.set_shift(True)
        self._keep = []          # host/device sources that must outlive async copies
        self._finished = False
        # what "auto" resolved to: "tc" (tcgen05 3xTF32) or "simt" (FFMA / DFMA)
        self.precision = "tc" if self.lib.spca_sketch_precision(self.h) == _PRECISIONS["tc"] else "simt"

    def set_shift(self, on: bool = True) -> None:
        """Column shift (spca_sketch_set_shift): accumulate A - 1 c^T, c = the
        mean of the pass's first (up to 256) rows, and restore the sketch of A in fp64 at finish.
        Before the first push of a pass; exclusive with normalisation."""
        _lib.check(self.lib.spca_sketch_set_shift(self.h, 1 if on else 0), self.h)

    def set_left(self, left) -> None:
        """Co-sketch operand L (m x l float64, numpy or CUDA tensor): the pass
        then accumulates H += A_i^T L[rows of A_i] in place of A_i^T G_i
        (spca_sketch_set_left) — legacy_single_pass's Yt and basic_rand_svd's
        B^T. ``None`` restores the plain sketch. Before the first push."""
        torch = torch_mod()
        if left is None:
            _lib.check(self.lib.spca_sketch_set_left(self.h, None, 0, _lib.MEM_DEVICE), self.h)
            return
        if is_torch(left):
            t = left.to(device=self.device, dtype=torch.float64).contiguous()
            if t.dim() != 2 or t.shape[1] != self.l:
                raise StreamFormatError(f"left operand has shape {tuple(t.shape)}, expected (*, {self.l})")
            _lib.check(self.lib.spca_sketch_set_left(self.h, ctypes.c_void_p(t.data_ptr()), int(t.shape[0]),
                                                     _lib.MEM_DEVICE), self.h)
            self._left = t  # the conversion kernel reads it in stream order
        else:
            a = np.ascontiguousarray(np.asarray(left, dtype=np.float64))
            if a.ndim != 2 or a.shape[1] != self.l:
                raise StreamFormatError(f"left operand has shape {a.shape}, expected (*, {self.l})")
            _lib.check(self.lib.spca_sketch_set_left(self.h, ctypes.c_void_p(a.ctypes.data), int(a.shape[0]),
                                                     _lib.MEM_PAGEABLE), self.h)

    # -- pushing ------------------------------------------------------------
    def push(self, values, first_row: int, final: bool = False) -> int:
        """Append one block; numpy (pageable host), pinned host tensor or CUDA tensor.
        ``final=True`` marks the last block of the stream: its trailing partial
        chunk is processed now instead of at finish (spca_sketch_push_final)."""
        torch = torch_mod()
        if is_torch(values):
            t = values
            if t.dim() != 2 or t.shape[1] != self.n:
                raise StreamFormatError(
                    f"block at row {first_row} has shape {tuple(t.shape)}, expected (*, {self.n})")
            want = torch.float32 if self.dtype == np.float32 else torch.float64
            if t.dtype != want:
                t = t.to(want)
            if t.stride(1) != 1:
                t = t.contiguous()
            if t.is_cuda:
                if t.device != self.device:
                    t = t.to(self.device)
                where = _lib.MEM_DEVICE
            else:
                where = _lib.MEM_PINNED if t.is_pinned() else _lib.MEM_PAGEABLE
            rows, ld, ptr = int(t.shape[0]), int(t.stride(0)) if t.shape[0] > 1 else self.n, t.data_ptr()
            self._keep.append(t)
        else:
            a = np.asarray(values)
            if a.ndim != 2 or a.shape[1] != self.n:
                raise StreamFormatError(
                    f"block at row {first_row} has shape {a.shape}, expected (*, {self.n})")
            if a.dtype != self.dtype or a.strides[1] != a.itemsize:
                a = np.ascontiguousarray(a, dtype=self.dtype)
            rows = a.shape[0]
            ld = a.strides[0] // a.itemsize if rows > 1 else self.n
            ptr = a.ctypes.data
            where = _lib.MEM_PAGEABLE
        if rows == 0 and not final:
            return 0
        fn = self.lib.spca_sketch_push_final if final else self.lib.spca_sketch_push
        _lib.check(fn(self.h, ctypes.c_void_p(ptr) if rows else None, rows, max(ld, self.n),
                      int(first_row), where), self.h)
        return rows

    def reset(self) -> None:
        """New pass, same Omega and allocations (spca_sketch_reset)."""
        _lib.check(self.lib.spca_sketch_reset(self.h), self.h)
        self._keep.clear()
        self._finished = False

    def sync(self) -> None:
        _lib.check(self.lib.spca_sketch_sync(self.h), self.h)
        self._keep.clear()

    # -- results ------------------------------------------------------------
    def finish(self, on_device: bool = True):
        """(g, h, col_sums, rows_seen) as CUDA float64 tensors (or numpy,
        read back through page-locked staging)."""
        torch = torch_mod()
        if not on_device:
            g, hh, cs, m = self.finish(on_device=True)
            return host_copy(g), host_copy(hh), host_copy(cs), m
        rows = ctypes.c_int64(0)
        _lib.check(self.lib.spca_sketch_rows(self.h, ctypes.byref(rows)), self.h)
        m = rows.value
        if on_device:
            g = torch.empty((m, self.l), dtype=torch.float64, device=self.device)
            hh = torch.empty((self.n, self.l), dtype=torch.float64, device=self.device)
            cs = torch.empty((self.n,), dtype=torch.float64, device=self.device)
            ptrs = (g.data_ptr() if m else None, hh.data_ptr(), cs.data_ptr())
            where = _lib.MEM_DEVICE
        else:
            g = np.empty((m, self.l))
            hh = np.empty((self.n, self.l))
            cs = np.empty(self.n)
            ptrs = (g.ctypes.data if m else None, hh.ctypes.data, cs.ctypes.data)
            where = _lib.MEM_PAGEABLE
        # the handle's stream must see torch's allocations (same stream here)
        rc = self.lib.spca_sketch_finish(self.h, *(ctypes.c_void_p(p) if p else None for p in ptrs),
                                         ctypes.byref(rows), where)
        self._keep.clear()
        _lib.check(rc, self.h)
        self._finished = True
        return g, hh, cs, m

    def omega_used(self, on_device: bool = True):
        """Omega exactly as the pass used it (n x l float64; fp32-rounded for
        fp32 data), copied from the device (spca_omega_used)."""
        torch = torch_mod()
        if on_device:
            out = torch.empty((self.n, self.l), dtype=torch.float64, device=self.device)
            _lib.check(self.lib.spca_omega_used(self.h, ctypes.c_void_p(out.data_ptr()), _lib.MEM_DEVICE), self.h)
            return out
        out = np.empty((self.n, self.l))
        _lib.check(self.lib.spca_omega_used(self.h, ctypes.c_void_p(out.ctypes.data), _lib.MEM_PAGEABLE), self.h)
        return out

    def allreduce_nccl(self, comm) -> int:
        """spca_allreduce: sum the finished [H | col_sums] over the ranks of an
        ncclComm_t (an integer pointer from the caller's NCCL) in place; returns
        the global row count. (torch.distributed callers use
        parallel.allreduce_sketch, which needs no raw communicator.)"""
        total = ctypes.c_int64(0)
        _lib.check(self.lib.spca_allreduce(self.h, ctypes.c_void_p(int(comm)), ctypes.byref(total)), self.h)
        return total.value

    def rows(self) -> int:
        """Rows pushed so far (spca_sketch_rows)."""
        r = ctypes.c_int64(0)
        _lib.check(self.lib.spca_sketch_rows(self.h, ctypes.byref(r)), self.h)
        return r.value

    def kernel_launches(self) -> int:
        return int(self.lib.spca_kernel_launches(self.h))

    def chunk_rows(self) -> int:
        return int(self.lib.spca_sketch_chunk_rows(self.h))

    def enable_timing(self, on: bool = True) -> None:
        _lib.check(self.lib.spca_enable_kernel_timing(self.h, 1 if on else 0), self.h)

    def kernel_time(self) -> tuple[float, int]:
        ms = ctypes.c_double(0)
        cnt = ctypes.c_int64(0)
        _lib.check(self.lib.spca_kernel_time_ms(self.h, ctypes.byref(ms), ctypes.byref(cnt)), self.h)
        return ms.value, cnt.value

    def close(self) -> None:
        if getattr(self, "h", None):
            self.lib.spca_sketch_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def run_pass(stream, omega, block_rows=None, compensated=False, precision="auto",
             device=None, keep=None, left=None, sk=None, shift=False):
    """Drive one traversal of ``stream`` through a GpuSketch; returns the
    finished GpuSketch (state still on the device). ``left`` sets a co-sketch
    operand (GpuSketch.set_left); ``sk`` reuses an open handle of the same
    shape for another traversal (reset first). ``shift`` turns on the column
    shift (spca_sketch_set_shift) — what the centered algorithms ask for, so
    post-hoc centering does not cancel fp32 rounding of a large mean."""
    om = omega if is_torch(omega) else np.asarray(omega)
    n, l = om.shape
    outer = stream
    src = stream.wrapped if isinstance(stream, PassCounter) else stream
    # NormalizedRowStream: the library normalizes the rows of the wrapped source
    # (fused into the pass on the tensor-core path); the raw source is pushed
    normalize = isinstance(src, NormalizedRowStream)
    if normalize:
        src = src.wrapped
    else:
        src = outer  # a PassCounter counts its own traversal
    dtype = np.dtype(getattr(src, "dtype", np.float64))
    if sk is None:
        sk = GpuSketch(n, om, dtype, precision=precision, device=device,
                       rows_hint=src.n_rows or 0, compensated=compensated, normalize=normalize,
                       shift=shift and not normalize)
    else:
        sk.reset()
    if left is not None:
        sk.set_left(left)
    fs = _file_source(src)
    if fs is not None:
        _push_file(sk, fs)
        for pc in {id(x): x for x in (src, outer) if isinstance(x, PassCounter)}.values():
            _count_pass(pc, sk)
    else:
        _push_source(sk, src, block_rows, n, l)
        if normalize and isinstance(outer, PassCounter):
            _count_pass(outer, sk)
    return sk


def _count_pass(pc: PassCounter, sk: "GpuSketch") -> None:
    pc.rows_read += int(sk.rows())
    pc.passes_completed += 1
    pc.pass_in_progress = False


def _push_source(sk: "GpuSketch", stream, block_rows, n: int, l: int) -> None:
    """Whole in-memory / device / pinned sources in one push (the library
    re-chunks canonically), anything else block by block as it arrives."""
    if has_whole(stream):
        kind, mat = stream.whole()
        if mat.shape[0]:
            sk.push(mat, 0, final=True)
        return
    if block_rows is None:
        block_rows = l
    # blocks are pushed as they come (a stream may reuse its block buffer,
    # so no look-ahead); the trailing partial chunk is flushed at finish
    for block in stream.blocks(block_rows):
        vals = block.values
        if getattr(vals, "ndim", None) != 2 or vals.shape[1] != n:
            raise StreamFormatError(
                f"block at row {block.first_row_index} has shape {tuple(vals.shape)}, "
                f"expected (*, {n})")
        sk.push(vals, block.first_row_index)


def _file_source(stream) -> Optional[FileRowStream]:
    inner = stream.wrapped if isinstance(stream, PassCounter) else stream
    return inner if isinstance(inner, FileRowStream) else None


def _push_file(sk: GpuSketch, fs: FileRowStream, nbuf: int = 3) -> None:
    """Stream a matrix file through page-locked buffers: a reader thread fills
    buffer j % nbuf with parallel positional reads (no host-side copy, the
    file's element type kept) while the library copies and sketches the
    previous ones; a buffer is refilled only after the event recorded behind
    its push on the sketch stream has completed."""
    torch = torch_mod()
    lay = fs.layout
    m, n = lay.rows, lay.cols
    tdt = torch.float32 if fs.dtype == np.float32 else torch.float64
    buf_rows = max(1, min(m, fs.buffer_bytes // lay.row_bytes))
    starts = list(range(0, m, buf_rows))
    nb = max(1, min(nbuf, len(starts)))
    bufs = [torch.empty((buf_rows, n), dtype=tdt, pin_memory=True) for _ in range(nb)]
    views = [b.numpy() for b in bufs]
    full: queue.Queue = queue.Queue()
    released: queue.Queue = queue.Queue()

    def reader():
        try:
            with ThreadPoolExecutor(fs.read_threads) as pool:
                for j, start in enumerate(starts):
                    i = j % nb
                    if j >= nb:
                        ri, ev = released.get()
                        if ri is None:  # the consumer gave up
                            return
                        ev.synchronize()
                    rows = min(buf_rows, m - start)
                    fs.read_rows_into(views[i], start, rows, pool)
                    full.put((i, start, rows))
            full.put(None)
        except BaseException as exc:  # handed to the consumer
            full.put(exc)

    th = threading.Thread(target=reader, name="spca-file-reader", daemon=True)
    th.start()
    try:
        while True:
            item = full.get()
            if item is None:
                break
            if isinstance(item, BaseException):
                raise item
            i, start, rows = item
            sk.push(bufs[i][:rows], start, final=start + rows == m)
            ev = torch.cuda.Event()
            ev.record(sk.stream)
            released.put((i, ev))
    except BaseException:
        released.put((None, None))
        raise
    finally:
        th.join(timeout=60)
    if m == 0:
        sk.push(np.empty((0, n), dtype=fs.dtype), 0, final=True)


def normalize_rows_device(t, out=None):
    """Rows of a CUDA tensor (float32/float64) to zero mean and unit norm with
    the libspca kernel (spca_normalize_rows), on torch's current stream.
    ``out`` (same shape and dtype, may be ``t``) receives the result."""
    torch = torch_mod()
    lib = _lib.load()
    if t.dim() != 2 or t.dtype not in (torch.float32, torch.float64) or not t.is_cuda:
        raise StreamFormatError("normalize_rows_device needs a 2-d float32/float64 CUDA tensor")
    if t.stride(1) != 1:
        t = t.contiguous()
    if out is None:
        out = torch.empty(t.shape, dtype=t.dtype, device=t.device)
    rows, n = int(t.shape[0]), int(t.shape[1])
    code = _lib.SPCA_F32 if t.dtype == torch.float32 else _lib.SPCA_F64
    st = torch.cuda.current_stream(t.device).cuda_stream
    with torch.cuda.device(t.device):
        rc = lib.spca_normalize_rows(ctypes.c_void_p(t.data_ptr()), rows, n, max(int(t.stride(0)), n),
                                     ctypes.c_void_p(out.data_ptr()), max(int(out.stride(0)), n), code,
                                     ctypes.c_void_p(st))
    _lib.check(rc)
    return out


def normalize_rows(block, device=None):
    """Shift each row to zero mean, then scale it to unit Euclidean norm; a
    constant row becomes the zero row (sketch.py:142-153). RowBlock or bare
    2-d array in, the same kind out; host input gives float64 numpy (as the
    reference), CUDA tensors stay on the device in their dtype. The
    arithmetic runs on the GPU (fp64)."""
    torch = torch_mod()
    bare = not isinstance(block, RowBlock)
    vals = block if bare else block.values
    if is_torch(vals) and vals.is_cuda:
        out = normalize_rows_device(vals)
    else:
        arr = np.ascontiguousarray(np.asarray(vals.cpu().numpy() if is_torch(vals) else vals,
                                              dtype=np.float64))
        if arr.ndim != 2:
            raise StreamFormatError("normalize_rows expects a 2-d block")
        if arr.shape[0] == 0 or arr.shape[1] == 0:
            out = arr.copy()
        else:
            dev = default_device(device)
            out = normalize_rows_device(torch.from_numpy(arr).to(dev)).cpu().numpy()
    return out if bare else RowBlock(block.first_row_index, out)


class NormalizedRowStream(RowStream):
    """View of a stream with normalize_rows applied to every block
    (sketch.py:156-182). ``blocks`` yields float64 numpy blocks like the
    reference; the device pass instead pushes the wrapped source unchanged
    and lets the library normalize (spca_sketch_set_normalize: fused into the
    pass kernel on the tensor-core path, a per-chunk workspace on the SIMT
    path), in the wrapped stream's element type."""

    def __init__(self, wrapped):
        self._wrapped = wrapped

    @property
    def wrapped(self):
        return self._wrapped

    @property
    def n_rows(self):
        return self._wrapped.n_rows

    @property
    def n_cols(self) -> int:
        return self._wrapped.n_cols

    @property
    def resettable(self) -> bool:
        return self._wrapped.resettable

    @property
    def dtype(self) -> np.dtype:
        return np.dtype(getattr(self._wrapped, "dtype", np.float64))

    def blocks(self, block_rows: int):
        for block in self._wrapped.blocks(block_rows):
            yield normalize_rows(block)


def sketch_pass(
    stream,
    omega: np.ndarray,
    block_rows: Optional[int] = None,
    fixed_order: bool = False,
    compensated: bool = False,
    *,
    precision: str = "auto",
    device=None,
    keep_on_device: bool = False,
    shift: bool = False,
) -> SketchState:
    """Accumulate the sketch of the streamed matrix in exactly one pass
    (sketch.py:52-116), on the GPU.

    ``block_rows`` defaults to l and is what a generic stream is asked for
    (sketch.py:76-77). ``fixed_order`` is accepted for signature parity: the
    device path is always order-fixed — bitwise identical for every block
    size and run to run — which is the property fixed_order buys on the CPU.
    ``compensated`` enables Kahan summation of col_sums across chunks.
    ``shift`` accumulates A - 1 c^T (c = the mean of the first rows) and adds the shift
    back in fp64: same results, fp32 accumulators sized by A's spread rather
    than its mean (the centered algorithms turn it on)."""
    om = omega if is_torch(omega) else np.asarray(omega, dtype=np.float64)
    if om.ndim != 2:
        raise StreamFormatError("omega must be 2-d")
    n, l = om.shape
    if stream.n_cols != n:
        raise StreamFormatError(f"stream has {stream.n_cols} columns but omega has {n} rows")
    sk = run_pass(stream, om, block_rows=block_rows, compensated=compensated,
                  precision=precision, device=device, shift=shift)
    try:
        g, h, cs, m = sk.finish(on_device=keep_on_device)
        used = sk.omega_used(on_device=keep_on_device)  # the library's copy: no host re-rounding
    finally:
        sk.close()
    return SketchState(g=g, h=h, col_sums=cs, rows_seen=int(m), omega=used)


def center_correct(state: SketchState, omega) -> SketchState:
    """Rewrite the sketch as if A had been column-centered (sketch.py:119-139):
    mu = col_sums/m, G -= 1 (mu^T Omega), H -= mu (1^T G); on the GPU in fp64.
    Returns the same array kind (numpy or CUDA tensor) it was given."""
    torch = torch_mod()
    if state.rows_seen == 0:
        raise EmptyStreamError("cannot center a sketch of zero rows")
    on_dev = is_torch(state.g)
    dev = state.g.device if on_dev else default_device()
    g = to_device64(state.g, dev)
    h = to_device64(state.h, dev)
    cs = to_device64(state.col_sums, dev)
    om = to_device64(omega, dev)
    mu = cs / state.rows_seen
    g_c = g - (mu @ om)[None, :]
    h_c = h - torch.outer(mu, g.sum(dim=0))
    z = torch.zeros_like(cs)
    if not on_dev:
        g_c, h_c, z = host_copy(g_c), host_copy(h_c), host_copy(z)
    return replace(state, g=g_c, h=h_c, col_sums=z)
