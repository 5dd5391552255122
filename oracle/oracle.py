"""CPU oracle for the FaSTED epsilon self-join -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import this module, and
only as the checker / the timed CPU baseline.  The product package
(``paper_2508_21230_b200``) never imports it: its path fails loudly when the
CUDA library is missing instead of falling back here.

Two restatements of the reference arithmetic (``/root/reference/pkg/src/mpjoin``):

* ``liboracle.so`` (``fasted_oracle.c``): FP32->FP16 RNE cast, RZ norms, the
  RZ-accumulated tiled join and a per-pair dist_sq evaluator.  Fast enough
  for the 16K x 128 oracle config and for sampled row blocks of the 1M-point
  configs.
* the numpy functions below (``add_rz``, ``combine_distance``,
  ``join_numpy``), which restate ``mma.add_rz`` (mma.py:45-64),
  ``mma.combine_distance`` (mma.py:143-157) and
  ``oracle.reference_mixed_scalar`` (oracle.py:67-108) op for op; they
  cross-check the C library on small inputs.

Parity is pinned by ``tests/golden/`` (vectors made by the reference itself,
see ``tests/golden/make_golden.py``) -- ``tests/test_oracle.py``.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None


def build() -> str:
    """Compile liboracle.so with the committed Makefile (gcc only)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        src = os.path.join(_HERE, "fasted_oracle.c")
        if not os.path.exists(_LIB_PATH) or (
            os.path.exists(src) and os.path.getmtime(src) > os.path.getmtime(_LIB_PATH)
        ):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        i64, p = ctypes.c_int64, ctypes.c_void_p
        L.oracle_f32_to_f16.restype = ctypes.c_uint16
        L.oracle_f32_to_f16.argtypes = [ctypes.c_float]
        L.oracle_f16_to_f32.restype = ctypes.c_float
        L.oracle_f16_to_f32.argtypes = [ctypes.c_uint16]
        L.oracle_to_half.restype = ctypes.c_int
        L.oracle_to_half.argtypes = [p, i64, i64, p, i64, i64, p, p]
        L.oracle_norms.restype = None
        L.oracle_norms.argtypes = [p, i64, i64, p]
        L.oracle_join.restype = i64
        L.oracle_join.argtypes = [p, p, i64, i64, i64, i64, i64, i64, i64,
                                  ctypes.c_float, ctypes.c_int, p, p, p, i64]
        L.oracle_pair_d2.restype = None
        L.oracle_pair_d2.argtypes = [p, p, i64, i64, p, p, p]
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


# ── to_half / norms (dataset.py:152-193) ────────────────────────────────


def to_half(values: np.ndarray, block_side: int = 128, kslice: int = 16):
    """(values16[n_pad, d_pad] float16, norms[n_pad] float32, first_overflow).

    first_overflow is the row-major flat index of the first coordinate whose
    FP16 cast overflowed (the point / dimension the reference's RangeError
    names, dataset.py:177-183), or -1.
    """
    x = np.ascontiguousarray(values, dtype=np.float32)
    n, d = x.shape
    n_pad = -(-n // block_side) * block_side
    d_pad = -(-d // kslice) * kslice
    out = np.zeros((n_pad, d_pad), dtype=np.uint16)
    norms = np.zeros(n_pad, dtype=np.float32)
    first = ctypes.c_int64(-1)
    rc = lib().oracle_to_half(_ptr(x), n, d, _ptr(out), n_pad, d_pad, _ptr(norms),
                              ctypes.byref(first))
    return out.view(np.float16), norms, int(first.value) if rc else -1


def norms_rz(values16: np.ndarray) -> np.ndarray:
    v = np.ascontiguousarray(values16).view(np.uint16)
    out = np.zeros(v.shape[0], dtype=np.float32)
    lib().oracle_norms(_ptr(v), v.shape[0], v.shape[1], _ptr(out))
    return out


# ── join (tiling.py:199-359 / oracle.py:67-108) ─────────────────────────


def eps_sq_of(epsilon: float) -> np.float32:
    """eps32 = f32(eps); eps_sq = f32(eps32 * eps32) (tiling.py:304-305)."""
    e32 = np.float32(epsilon)
    return np.float32(e32 * e32)


def join(values16: np.ndarray, norms: np.ndarray, n_logical: int, epsilon: float,
         rows=None, cols=None, threads: int | None = None, count_only: bool = False,
         capacity: int | None = None):
    """Reference pairs (i, j, dist_sq) over rows x cols, canonical order.

    rows / cols are (begin, end) 0-based point ranges (default: everything).
    Returns (i uint32, j uint32, d float32) or, with count_only, the count.
    """
    v = np.ascontiguousarray(values16).view(np.uint16)
    s = np.ascontiguousarray(norms, dtype=np.float32)
    n_pad, d_pad = v.shape
    r0, r1 = rows if rows is not None else (0, n_pad)
    c0, c1 = cols if cols is not None else (0, n_pad)
    if threads is None:
        threads = len(os.sched_getaffinity(0))
    es = eps_sq_of(epsilon)
    L = lib()
    if count_only:
        cnt = L.oracle_join(_ptr(v), _ptr(s), n_logical, n_pad, d_pad, r0, r1, c0, c1,
                            float(es), threads, None, None, None, 0)
        if cnt < 0:
            raise MemoryError("oracle_join failed")
        return int(cnt)
    if capacity is None:
        capacity = L.oracle_join(_ptr(v), _ptr(s), n_logical, n_pad, d_pad, r0, r1, c0, c1,
                                 float(es), threads, None, None, None, 0)
    cap = max(int(capacity), 1)
    oi = np.empty(cap, np.uint32)
    oj = np.empty(cap, np.uint32)
    od = np.empty(cap, np.float32)
    cnt = L.oracle_join(_ptr(v), _ptr(s), n_logical, n_pad, d_pad, r0, r1, c0, c1,
                        float(es), threads, _ptr(oi), _ptr(oj), _ptr(od), cap)
    if cnt < 0:
        raise MemoryError("oracle_join failed")
    k = min(int(cnt), cap)
    return oi[:k], oj[:k], od[:k]


def pair_d2(values16: np.ndarray, norms: np.ndarray, i: np.ndarray, j: np.ndarray) -> np.ndarray:
    """Reference dist_sq (clamped) for explicit 1-based pairs."""
    v = np.ascontiguousarray(values16).view(np.uint16)
    s = np.ascontiguousarray(norms, dtype=np.float32)
    i = np.ascontiguousarray(i, dtype=np.uint32)
    j = np.ascontiguousarray(j, dtype=np.uint32)
    out = np.empty(i.shape[0], np.float32)
    lib().oracle_pair_d2(_ptr(v), _ptr(s), v.shape[1], i.shape[0], _ptr(i), _ptr(j), _ptr(out))
    return out


# ── numpy restatements (cross-check of the C library on small inputs) ───


def add_rz(a, b):
    """FP32 add rounded toward zero via FP64 2Sum (mma.py:45-64)."""
    a64 = np.asarray(a, dtype=np.float64)
    b64 = np.asarray(b, dtype=np.float64)
    s = a64 + b64
    bb = s - a64
    err = (a64 - (s - bb)) + (b64 - bb)
    r = s.astype(np.float32)
    t = (s - r.astype(np.float64)) + err
    step = ((r > 0) & (t < 0)) | ((r < 0) & (t > 0))
    return np.where(step, np.nextafter(r, np.float32(0.0)), r).astype(np.float32)


def combine_distance(a, s_i, s_j):
    """max(((-2 a) + s_i) + s_j, 0) in FP32 round-to-nearest (mma.py:143-157)."""
    d2 = (np.float32(-2.0) * np.asarray(a, np.float32) + np.asarray(s_i, np.float32)) \
        + np.asarray(s_j, np.float32)
    return np.maximum(d2, np.float32(0.0))


def join_numpy(values16: np.ndarray, norms: np.ndarray, n_logical: int, epsilon: float):
    """Untiled order-exact join (oracle.py:67-108), small n only."""
    wide = np.asarray(values16, dtype=np.float32)
    n_pad = wide.shape[0]
    es = eps_sq_of(epsilon)
    acc = np.zeros((n_logical, n_pad), np.float32)
    for k in range(wide.shape[1]):
        acc = add_rz(acc, wide[:n_logical, k][:, None] * wide[:, k][None, :])
    d2 = combine_distance(acc, norms[:n_logical][:, None], norms[None, :])
    keep = d2 <= es
    keep[:, n_logical:] = False
    rr, cc = np.nonzero(keep)
    return (rr + 1).astype(np.uint32), (cc + 1).astype(np.uint32), d2[rr, cc]


# ── pairs payload (cli.py:54,72-77) ─────────────────────────────────────

PAIR_DTYPE = np.dtype([("i", "<u4"), ("j", "<u4"), ("dist_sq", "<f4")])


def pairs_payload(i, j, d) -> bytes:
    rec = np.empty(len(i), dtype=PAIR_DTYPE)
    rec["i"] = i
    rec["j"] = j
    rec["dist_sq"] = np.asarray(d, np.float32)
    return np.uint64(len(i)).tobytes() + rec.tobytes()
