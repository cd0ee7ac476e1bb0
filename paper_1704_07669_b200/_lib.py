"""ctypes binding of libspca.so (include/spca.h).

The product path has no CPU fallback: if the shared library or a CUDA
device is missing, every entry point raises ``DeviceError``.
"""

from __future__ import annotations

import ctypes
import os
import threading
from ctypes import POINTER, c_char_p, c_double, c_int, c_int64, c_size_t, c_void_p

from .errors import (
    CapabilityError,
    ConfigError,
    DataError,
    DeviceError,
    DeviceMemoryError,
    EmptyStreamError,
    StreamFormatError,
)

HERE = os.path.dirname(os.path.abspath(__file__))
# SPCA_LIB: load a differently-built copy (A/B timing of build variants)
LIB_PATH = os.environ.get("SPCA_LIB") or os.path.join(HERE, "libspca.so")

SPCA_F32, SPCA_F64 = 0, 1
PREC_AUTO, PREC_SIMT, PREC_TC = 0, 1, 2
MEM_DEVICE, MEM_PINNED, MEM_PAGEABLE = 0, 1, 2

OK, ERR_FORMAT, ERR_DATA, ERR_CAPABILITY, ERR_CONFIG, ERR_CUDA, ERR_OOM, ERR_STATE, ERR_EMPTY = range(9)

# every symbol include/spca.h declares, with (restype, argtypes)
SIGNATURES = {
    "spca_abi_version": (c_int, []),
    "spca_build_info": (c_char_p, []),
    "spca_sketch_create": (c_int, [POINTER(c_void_p), c_int64, c_int64, c_int, c_int, c_void_p,
                                   c_int, c_int, c_void_p, c_int64, c_int]),
    "spca_sketch_push": (c_int, [c_void_p, c_void_p, c_int64, c_int64, c_int64, c_int]),
    "spca_sketch_push_final": (c_int, [c_void_p, c_void_p, c_int64, c_int64, c_int64, c_int]),
    "spca_sketch_precision": (c_int, [c_void_p]),
    "spca_sketch_reset": (c_int, [c_void_p]),
    "spca_sketch_sync": (c_int, [c_void_p]),
    "spca_sketch_rows": (c_int, [c_void_p, POINTER(c_int64)]),
    "spca_sketch_chunk_rows": (c_int64, [c_void_p]),
    "spca_sketch_finish": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, POINTER(c_int64), c_int]),
    "spca_device_views": (c_int, [c_void_p, POINTER(c_void_p), POINTER(c_void_p)]),
    "spca_center_correct": (c_int, [c_void_p, c_int64, c_void_p, c_void_p, c_int]),
    "spca_g_colsum": (c_int, [c_void_p, c_void_p, c_int]),
    "spca_sketch_set_normalize": (c_int, [c_void_p, c_int]),
    "spca_sketch_set_left": (c_int, [c_void_p, c_void_p, c_int64, c_int]),
    "spca_sketch_set_shift": (c_int, [c_void_p, c_int]),
    "spca_omega_used": (c_int, [c_void_p, c_void_p, c_int]),
    "spca_allreduce": (c_int, [c_void_p, c_void_p, POINTER(c_int64)]),
    "spca_normalize_rows": (c_int, [c_void_p, c_int64, c_int64, c_int64, c_void_p, c_int64, c_int, c_void_p]),
    "spca_qb_workspace_elems": (c_int64, [c_int64, c_int, c_int]),
    "spca_qb_block": (c_int, [c_int64, c_int, c_int, c_void_p, c_int64, c_void_p, c_int64, c_void_p, c_void_p,
                              c_void_p, c_int64, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    "spca_gaussian_device": (c_int, [c_void_p, c_int64, ctypes.c_uint64, ctypes.c_uint64, c_void_p, c_void_p,
                                     c_void_p, c_double, c_double, c_void_p]),
    "spca_qb_omega_proj_ws": (c_int64, [c_int64, c_int, c_int]),
    "spca_qb_omega_proj": (c_int, [c_int64, c_int, c_int, c_void_p, c_int64, c_void_p, c_int64, c_void_p, c_void_p,
                                   c_int64, c_void_p]),
    "spca_qb_b_rows": (c_int, [c_int64, c_int, c_int, c_void_p, c_int64, c_void_p, c_int64, c_void_p, c_void_p,
                               c_void_p, c_void_p, c_void_p]),
    "spca_last_error": (c_int, [c_void_p, POINTER(c_int), POINTER(c_int64), c_char_p, c_size_t]),
    "spca_kernel_launches": (c_int64, [c_void_p]),
    "spca_enable_kernel_timing": (c_int, [c_void_p, c_int]),
    "spca_kernel_time_ms": (c_int, [c_void_p, POINTER(c_double), POINTER(c_int64)]),
    "spca_sketch_destroy": (None, [c_void_p]),
}

_lib = None
_lock = threading.Lock()


def load(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load libspca.so and bind every declared symbol (fails loudly)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise DeviceError(
                f"{path} is missing: build it with `python -m paper_1704_07669_b200.build` "
                "(there is no CPU fallback for the sketch pass)")
        lib = ctypes.CDLL(path)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if lib.spca_abi_version() != 1:
            raise DeviceError("libspca ABI version mismatch")
        _lib = lib
        return lib


def last_error(handle=None) -> tuple[int, int, str]:
    lib = load()
    code = c_int(0)
    row = c_int64(-1)
    buf = ctypes.create_string_buffer(512)
    lib.spca_last_error(handle, ctypes.byref(code), ctypes.byref(row), buf, 512)
    return code.value, row.value, buf.value.decode(errors="replace")


def check(rc: int, handle=None) -> None:
    """Map a status code onto the reference's exception classes."""
    if rc == OK:
        return
    code, row, msg = last_error(handle)
    if code == OK:
        code = rc
    if code == ERR_FORMAT:
        raise StreamFormatError(msg)
    if code == ERR_DATA:
        raise DataError(msg, row=row if row >= 0 else None)
    if code == ERR_CAPABILITY:
        raise CapabilityError(msg)
    if code == ERR_CONFIG:
        raise ConfigError(msg)
    if code == ERR_EMPTY:
        raise EmptyStreamError(msg)
    if code == ERR_OOM:
        raise DeviceMemoryError(msg)
    raise DeviceError(msg or f"libspca error {code}")
