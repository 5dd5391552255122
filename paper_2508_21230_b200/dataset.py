"""Point datasets, synthesis, and the GPU FP16 conversion (drop-in for
/root/reference/pkg/src/mpjoin/dataset.py).

``to_half`` and ``compute_squared_norms`` run on the GPU (kernel 1,
``csrc/quantize.cu``) and return the reference's host types with the same
bits: FP16 round-to-nearest-even values, zero padded to
``[n_pad, d_pad]``, and FP32 squared norms accumulated round-toward-zero in
ascending k (dataset.py:152-193, _kernel.py:79-93).  The device copies are
kept on the returned ``HalfDataset`` so ``self_join`` does not upload them
again.
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .errors import ArgumentError, FormatError, RangeError

__all__ = [
    "Dataset",
    "HalfDataset",
    "load_fvecs",
    "generate_synthetic",
    "synthetic_rows",
    "to_half",
    "compute_squared_norms",
]

DEFAULT_BLOCK_SIDE = 128
DEFAULT_KSLICE = 16
FP16_MAX = 65504.0


@dataclass(frozen=True)
class Dataset:
    """n x d row-major matrix of finite FP32 coordinates, n >= 1, d >= 1
    (dataset.py:39-62)."""

    values: np.ndarray

    def __post_init__(self):
        arr = np.ascontiguousarray(self.values, dtype=np.float32)
        if arr.ndim != 2:
            raise ArgumentError(f"values must be 2-D, got shape {arr.shape}")
        if arr.shape[0] < 1 or arr.shape[1] < 1:
            raise ArgumentError(f"dataset must have n >= 1 and d >= 1, got {arr.shape}")
        if not np.isfinite(arr).all():
            i, k = np.argwhere(~np.isfinite(arr))[0]
            raise ArgumentError(f"non-finite coordinate at point {i}, dimension {k}")
        object.__setattr__(self, "values", arr)

    @property
    def n(self) -> int:
        return self.values.shape[0]

    @property
    def d(self) -> int:
        return self.values.shape[1]


@dataclass(frozen=True)
class HalfDataset:
    """Zero-padded FP16 working copy plus FP32 RZ squared norms
    (dataset.py:65-86).  ``device_cache`` maps a CUDA device index to the
    resident (values, norms) tensors; ``count_memo`` holds the engine's last
    exact pair count per (epsilon, range, kernel) so repeated joins of this
    dataset size their buffers once.  Neither takes part in equality."""

    n_logical: int
    d_logical: int
    values: np.ndarray  # (n_padded, d_padded) float16
    norms: np.ndarray   # (n_padded,) float32
    device_cache: dict = field(default_factory=dict, compare=False, repr=False)
    count_memo: dict = field(default_factory=dict, compare=False, repr=False)

    @property
    def n_padded(self) -> int:
        return self.values.shape[0]

    @property
    def d_padded(self) -> int:
        return self.values.shape[1]


def load_fvecs(path) -> Dataset:
    """Read an fvecs file (int32 dim header + dim float32 per record) with the
    reference's error reporting (dataset.py:89-132)."""
    with open(path, "rb") as f:
        raw = f.read()
    size = len(raw)
    name = os.fspath(path)
    if size == 0:
        raise FormatError(f"{name}: empty file, a dataset needs n >= 1")
    if size < 4:
        raise FormatError(f"{name}: truncated dimension header at byte offset 0")
    d = int(np.frombuffer(raw, dtype="<i4", count=1)[0])
    if d <= 0:
        raise FormatError(f"{name}: dimension header {d} at byte offset 0 must be >= 1")
    stride = 4 + 4 * d
    n_full = size // stride
    if n_full:
        heads = np.frombuffer(raw, dtype="<i4", count=n_full * (1 + d)).reshape(n_full, 1 + d)[:, 0]
        bad = np.nonzero(heads != d)[0]
        if bad.size:
            raise FormatError(
                f"{name}: inconsistent dimension {int(heads[bad[0]])} (first record had {d}) "
                f"at byte offset {int(bad[0]) * stride}")
    if size % stride:
        off = n_full * stride
        raise FormatError(
            f"{name}: truncated record at byte offset {off} "
            f"({size - off} bytes left, record needs {stride})")
    values = np.frombuffer(raw, dtype="<f4").reshape(n_full, 1 + d)[:, 1:]
    return Dataset(values.astype(np.float32))


def generate_synthetic(n: int, d: int, seed: int, lo: float = 0.0, hi: float = 1.0) -> Dataset:
    """i.i.d. uniform [lo, hi) coordinates, bit-identical to the reference's
    generator (dataset.py:135-149: PCG64 ``random(float32)`` scaled)."""
    if n < 1 or d < 1:
        raise ArgumentError(f"need n >= 1 and d >= 1, got n={n}, d={d}")
    if not (lo < hi) or not np.isfinite(hi - lo):
        raise ArgumentError(f"need lo < hi with finite span, got [{lo}, {hi})")
    rng = np.random.default_rng(seed)
    unit = rng.random((n, d), dtype=np.float32)
    return Dataset(unit * np.float32(hi - lo) + np.float32(lo))


def synthetic_rows(n: int, d: int, seed: int, r0: int, r1: int, lo: float = 0.0,
                   hi: float = 1.0) -> np.ndarray:
    """Rows [r0, r1) of ``generate_synthetic(n, d, seed, lo, hi).values``
    without generating the rows before them (PCG64 ``advance``; a float32
    draw consumes half of one 64-bit output).  Lets tests and the bench
    sample tiles of the 5M x 384 shape cheaply."""
    if not (0 <= r0 <= r1 <= n):
        raise ArgumentError(f"row range [{r0}, {r1}) outside [0, {n})")
    rng = np.random.default_rng(seed)
    skip = r0 * d
    rng.bit_generator.advance(skip // 2)
    if skip % 2:
        rng.random(1, dtype=np.float32)
    unit = rng.random((r1 - r0, d), dtype=np.float32)
    return unit * np.float32(hi - lo) + np.float32(lo)


def _padded_shape(n: int, d: int, block_side: int, kslice: int):
    return -(-n // block_side) * block_side, -(-d // kslice) * kslice


def to_half(ds: Dataset, block_side: int = DEFAULT_BLOCK_SIDE, kslice: int = DEFAULT_KSLICE,
            device: int | None = None, keep_on_device: bool = True,
            pin_host: bool = False) -> HalfDataset:
    """FP16 (RNE) conversion, zero padding and RZ norms on the GPU.

    Same result bits and the same RangeError message as the reference
    (dataset.py:164-193).  ``pin_host`` returns the host arrays in pinned
    memory (fast later uploads).
    """
    import torch

    if block_side < 1 or kslice < 1:
        raise ArgumentError("block_side and kslice must be >= 1")
    if device is None:
        device = torch.cuda.current_device() if torch.cuda.is_available() else 0
    _lib.require_device(device)
    n, d = ds.n, ds.d
    n_pad, d_pad = _padded_shape(n, d, block_side, kslice)
    d_dev = -(-d_pad // 8) * 8  # kernel row pitch needs 16-byte rows
    L = _lib.load()
    with torch.cuda.device(device):
        stream = torch.cuda.current_stream()
        x = torch.from_numpy(ds.values).to(device=f"cuda:{device}", non_blocking=True)
        vals = torch.empty((n_pad, d_dev), dtype=torch.float16, device=f"cuda:{device}")
        norms = torch.empty(n_pad, dtype=torch.float32, device=f"cuda:{device}")
        first = ctypes.c_int64(-1)
        st = L.fasted_quantize(x.data_ptr(), n, d, vals.data_ptr(), n_pad, d_dev,
                               norms.data_ptr(), ctypes.byref(first), stream.cuda_stream)
        if st == _lib.ERR_RANGE:
            i, k = divmod(int(first.value), d)
            raise RangeError(
                f"coordinate {ds.values[i, k]!r} of point {i} (dimension {k}) "
                f"exceeds the FP16 range (max {FP16_MAX})")
        _lib.check(st, "fasted_quantize")
        del x
        host_vals = vals[:, :d_pad] if d_dev != d_pad else vals
        if pin_host:
            hv = torch.empty((n_pad, d_pad), dtype=torch.float16, pin_memory=True)
            hn = torch.empty(n_pad, dtype=torch.float32, pin_memory=True)
            hv.copy_(host_vals, non_blocking=True)
            hn.copy_(norms, non_blocking=True)
            stream.synchronize()
            values_np, norms_np = hv.numpy(), hn.numpy()
        else:
            values_np = host_vals.cpu().numpy()
            norms_np = norms.cpu().numpy()
    hd = HalfDataset(n_logical=n, d_logical=d, values=values_np, norms=norms_np)
    if keep_on_device and d_dev == d_pad:
        hd.device_cache[device] = (vals, norms)
    return hd


def compute_squared_norms(hd: HalfDataset, device: int | None = None) -> np.ndarray:
    """FP32 RZ squared norms of every (padded) point, on the GPU
    (dataset.py:159-161)."""
    import torch

    if device is None:
        device = torch.cuda.current_device() if torch.cuda.is_available() else 0
    _lib.require_device(device)
    n_pad, d_pad = hd.values.shape
    with torch.cuda.device(device):
        stream = torch.cuda.current_stream()
        v = torch.from_numpy(np.ascontiguousarray(hd.values)).to(f"cuda:{device}")
        out = torch.empty(n_pad, dtype=torch.float32, device=f"cuda:{device}")
        _lib.check(_lib.load().fasted_norms(v.data_ptr(), n_pad, d_pad, out.data_ptr(),
                                            stream.cuda_stream), "fasted_norms")
        return out.cpu().numpy()
