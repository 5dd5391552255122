"""ctypes binding of libfasted.so (the C ABI declared in include/fasted.h).

This is the seam a reference maintainer would add to mpjoin: the numba
backend (_kernel.py) is replaced by these calls.  There is no fallback --
if the library or an sm_100 GPU is missing, every entry point raises
:class:`DeviceError`.
"""

from __future__ import annotations

import ctypes
import os
import threading

from .errors import ArgumentError, CapacityError, DeviceError, RangeError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libfasted.so")
# Same sources built with -DFASTED_EXPERIMENTS (csrc/experiments.h): the
# environment overrides of the kernel-form choice, the diagnostic flags and
# the retired kernel forms.  Used by scripts/ and by the bit-identity tests
# only; the product path never loads it.
EXP_LIB_PATH = os.path.join(_HERE, "libfasted_exp.so")

OK, ERR_ARGUMENT, ERR_RANGE, ERR_CAPACITY, ERR_CUDA, ERR_UNSUPPORTED = 0, 2, 3, 4, 5, 6
JOIN_TC, JOIN_EXACT, JOIN_COUNT, JOIN_SYMMETRIC, JOIN_LOW_OUTPUT, JOIN_APPEND = 0, 1, 2, 4, 8, 16
JOIN_SPARSE = 32

# Every symbol include/fasted.h declares (tests check the .so exports them).
EXPORTS = (
    "fasted_abi_version", "fasted_strerror", "fasted_last_error", "fasted_device_check",
    "fasted_device_info", "fasted_join_kernel_name", "fasted_quantize", "fasted_quantize_async",
    "fasted_norms", "fasted_join",
    "fasted_sort_workspace_bytes", "fasted_sort_pairs", "fasted_fp64_rows",
)

_libs: dict = {}
_lock = threading.Lock()


def load():
    """Load and type the product library libfasted.so (no GPU needed)."""
    return _load(LIB_PATH)


def load_experimental():
    """Load libfasted_exp.so (experiments and bit-identity tests only)."""
    return _load(EXP_LIB_PATH)


def _load(path):
    with _lock:
        if path in _libs:
            return _libs[path]
        if not os.path.exists(path):
            raise DeviceError(
                f"{path} is not built; run `python __graft_entry__.py` (build()) first")
        L = ctypes.CDLL(path)
        i64, u64, p, ci, f = (ctypes.c_int64, ctypes.c_uint64, ctypes.c_void_p, ctypes.c_int,
                              ctypes.c_float)
        L.fasted_abi_version.restype = ci
        L.fasted_abi_version.argtypes = []
        L.fasted_strerror.restype = ctypes.c_char_p
        L.fasted_strerror.argtypes = [ci]
        L.fasted_last_error.restype = ctypes.c_char_p
        L.fasted_last_error.argtypes = []
        L.fasted_device_check.restype = ci
        L.fasted_device_check.argtypes = [ci]
        L.fasted_join_kernel_name.restype = ctypes.c_char_p
        L.fasted_join_kernel_name.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ci]
        L.fasted_device_info.restype = ci
        L.fasted_device_info.argtypes = [ctypes.POINTER(ci), ctypes.c_char_p, ci]
        L.fasted_quantize.restype = ci
        L.fasted_quantize.argtypes = [p, i64, i64, p, i64, i64, p, ctypes.POINTER(i64), p]
        if hasattr(L, "fasted_quantize_async"):   # (older experiment builds lack it)
            L.fasted_quantize_async.restype = ci
            L.fasted_quantize_async.argtypes = [p, i64, i64, p, i64, i64, p, p, p]
        L.fasted_norms.restype = ci
        L.fasted_norms.argtypes = [p, i64, i64, p, p]
        L.fasted_join.restype = ci
        L.fasted_join.argtypes = [p, p, i64, i64, i64, i64, i64, i64, i64, f, ci,
                                  p, u64, p, p]
        L.fasted_sort_workspace_bytes.restype = ctypes.c_size_t
        L.fasted_sort_workspace_bytes.argtypes = [i64, i64]
        L.fasted_sort_pairs.restype = ci
        L.fasted_sort_pairs.argtypes = [p, u64, i64, i64, i64, p, p, p, p, ctypes.c_size_t,
                                        p, ctypes.c_size_t, p]
        L.fasted_fp64_rows.restype = ci
        L.fasted_fp64_rows.argtypes = [p, i64, i64, p, i64, ctypes.c_double, p, u64, p, p]
        if L.fasted_abi_version() != 2:
            raise DeviceError("libfasted ABI version mismatch")
        _libs[path] = L
        return L


def check(status: int, what: str, lib=None) -> None:
    """Map a C-ABI status to the reference's exception classes (`lib`: the
    library that returned it -- its thread-local last error -- default the
    product library)."""
    if status == OK:
        return
    L = lib if lib is not None else load()
    msg = (L.fasted_last_error() or b"").decode(errors="replace")
    text = f"{what}: {L.fasted_strerror(status).decode()}" + (f" ({msg})" if msg else "")
    if status == ERR_ARGUMENT:
        raise ArgumentError(text)
    if status == ERR_RANGE:
        raise RangeError(text)
    if status == ERR_CAPACITY:
        raise CapacityError(text)
    raise DeviceError(text)


_checked_devices: set = set()


def require_device(device: int) -> None:
    """Fail loudly unless `device` is an sm_100 GPU (called once per device)."""
    if device in _checked_devices:
        return
    import torch

    if not torch.cuda.is_available():
        raise DeviceError("no CUDA device: the FaSTED engine runs on B200 (sm_100a) only")
    with torch.cuda.device(device):
        check(load().fasted_device_check(device), f"device {device}")
    _checked_devices.add(device)
