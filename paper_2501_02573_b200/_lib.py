"""ctypes binding of ``lib/liblinattn_b200.so`` (C ABI: include/linattn_b200.h).

There is no fallback: if the library is missing, or CUDA is unavailable, every
call raises.  The library is built in-tree by ``make`` / ``__graft_entry__.build()``.
"""

from __future__ import annotations

import ctypes
import os

from .errors import LinAttnError, ParameterError, ResourceError, ShapeError, UsageError

LIB_PATH = os.environ.get("LINATTN_LIB") or os.path.join(
    os.path.dirname(os.path.abspath(__file__)), "lib", "liblinattn_b200.so")  # LINATTN_LIB: dev A/B builds

OK, ESHAPE, EPARAM, EDTYPE, EUNSUPPORTED, ECUDA, ENOMEM = range(7)
F32, BF16 = 0, 1
KERNEL_AUTO, KERNEL_TC, KERNEL_SIMT, KERNEL_TF32 = 0, 1, 2, 3
ABI_VERSION = 4

_lib = None

_i64 = ctypes.c_int64
_vp = ctypes.c_void_p
_SIGS = {
    "linattn_prefill": [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _i64, _i64, _i64, _i64,
                        ctypes.c_int, ctypes.c_int, _vp],
    "linattn_state_pass": [_vp, _vp, _vp, _vp, _i64, _i64, _i64, _i64, _i64, ctypes.c_int,
                           ctypes.c_int, _vp],
    "linattn_prefix_combine": [_vp, _vp, ctypes.POINTER(_i64), ctypes.c_int, ctypes.c_int, _vp,
                               _i64, _i64, _i64, _i64, _vp],
    "linattn_decode_step": [_vp, _vp, _vp, _vp, _vp, _vp, _i64, _i64, _i64, _i64, ctypes.c_int, _vp],
    "linattn_recurrent": [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _i64, _i64, _i64, _i64, ctypes.c_int, _vp],
    "linattn_prefill_kernel": [_i64, _i64, ctypes.c_int],
    "linattn_seq_plan": [_i64, _i64, _i64, _i64, _i64, ctypes.c_int, ctypes.c_int, ctypes.POINTER(_i64)],
    "linattn_state_pass_segmented": [_vp, _vp, _vp, _vp, _i64, _i64, _i64, _i64, _i64, ctypes.c_int,
                                     ctypes.c_int, _i64, _i64, _i64, _vp],
    "linattn_prefill_segmented": [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _i64, _i64, ctypes.c_int,
                                  _i64, _i64, _i64, _i64, _i64, ctypes.c_int, ctypes.c_int, _i64, _vp],
    "linattn_segment_prefix": [_vp, _i64, _i64, _i64, _vp, _i64, _i64, _vp, _i64, _i64, _i64, _i64, _i64, _vp],
    "linattn_state_at": [_vp, _i64, _i64, _i64, _vp, _vp, _i64, _vp, _i64, _i64, _i64, _i64, _i64, _vp],
    "linattn_nonfinite_index": [_vp, _i64, ctypes.c_int, _vp, _vp],
    "linattn_prefill_checked": [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _i64, _i64, _i64, _i64,
                                ctypes.c_int, ctypes.c_int, _vp, _vp],
    "linattn_release_workspace": [],
    "linattn_last_error": [],
    "linattn_abi_version": [],
    "linattn_launch_count": [],
}
EXPORTED = tuple(_SIGS)


def load(path: str = LIB_PATH):
    """Load (once) and return the ctypes library; raise LinAttnError if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise LinAttnError(
            f"CUDA extension not built: {path} is missing (run `make` or __graft_entry__.build())")
    lib = ctypes.CDLL(path)
    for name, args in _SIGS.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = ctypes.c_int
    lib.linattn_last_error.restype = ctypes.c_char_p
    lib.linattn_launch_count.restype = ctypes.c_int64
    if lib.linattn_abi_version() != ABI_VERSION:
        raise LinAttnError(f"ABI mismatch: library {lib.linattn_abi_version()} != {ABI_VERSION}")
    _lib = lib
    return lib


def check(status: int) -> None:
    """Map a C status onto the reference exception classes."""
    if status == OK:
        return
    msg = _lib.linattn_last_error().decode(errors="replace") if _lib is not None else ""
    if status == ESHAPE:
        raise ShapeError(msg)
    if status == EPARAM:
        raise ParameterError(msg)
    if status in (EDTYPE, EUNSUPPORTED):
        raise UsageError(msg)
    if status == ENOMEM:
        raise ResourceError(msg)
    raise LinAttnError(msg or f"linattn status {status}")


def launch_count() -> int:
    return int(load().linattn_launch_count())
