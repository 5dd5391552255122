"""Measurement and accuracy helpers (mirrors the hot-path-relevant part of
/root/reference/pkg/src/mpjoin/analysis.py) plus the band-parity
classifier used to state the tensor-core path's correctness contract.

Host-side numpy: these run on result sets, not inside the join.
"""

from __future__ import annotations

from collections import defaultdict
from dataclasses import dataclass

import numpy as np

from .errors import ArgumentError, CalibrationError
from .tiling import ResultSet

__all__ = [
    "selectivity", "derived_flops", "distance_tflops", "overlap_accuracy",
    "overlap_accuracy_sets", "ErrorStats",
    "distance_error_stats", "pairwise_sqdist_fp64", "brute_force_fp64_rows",
    "CalibrationResult", "calibrate_epsilon", "BandReport", "band_compare",
]

DEFAULT_ERROR_BINS = 61


def selectivity(rs: ResultSet) -> float:
    """Mean neighbours per point, (|R| - n) / n (analysis.py:222-226)."""
    if rs.n < 1:
        raise ArgumentError("result set must cover a dataset with n >= 1")
    return (len(rs) - rs.n) / rs.n


def derived_flops(n_padded: int, d_padded: int, elapsed_seconds: float) -> float:
    """Padded 2 n_pad^2 d_pad / t in TFLOPS (analysis.py:303-307)."""
    if elapsed_seconds <= 0:
        raise ArgumentError(f"elapsed_seconds must be > 0, got {elapsed_seconds}")
    return 2.0 * float(n_padded) ** 2 * float(d_padded) / elapsed_seconds / 1e12


def distance_tflops(n: int, d: int, elapsed_seconds: float) -> float:
    """Headline metric: logical 2 n^2 d / t in TFLOPS."""
    if elapsed_seconds <= 0:
        raise ArgumentError(f"elapsed_seconds must be > 0, got {elapsed_seconds}")
    return 2.0 * float(n) ** 2 * float(d) / elapsed_seconds / 1e12


def _neighbor_sets(rs: ResultSet) -> dict:
    sets: dict = defaultdict(set)
    for i, j in zip(rs.i.tolist(), rs.j.tolist()):
        sets[i].add(j)
    return sets


def overlap_accuracy(test: ResultSet, truth: ResultSet, points=None) -> float:
    """Eq. 3: mean per-point IoU of neighbour sets (analysis.py:127-147).
    ``points`` (1-based) restricts the mean to a row sample.

    Vectorised over the pair arrays (the reference builds one Python set per
    point, which takes minutes at 1M points): per point p, |A_p & B_p| from
    the sorted-key intersection, |A_p| and |B_p| from bincounts; a point with
    both sets empty scores 1, one side empty 0.  The per-point ratios are
    summed in ascending point order (np.cumsum is a sequential sum), the
    reference loop's order, so the result is bit-identical."""
    if test.n != truth.n:
        raise ArgumentError(f"result sets cover different datasets: n={test.n} vs n={truth.n}")
    n = int(test.n)
    tk = np.unique(_pair_keys(test.i, test.j))
    rk = np.unique(_pair_keys(truth.i, truth.j))
    common = np.intersect1d(tk, rk, assume_unique=True)
    row = lambda k: (k >> np.uint64(32)).astype(np.int64)  # noqa: E731
    na = np.bincount(row(tk), minlength=n + 1)
    nb = np.bincount(row(rk), minlength=n + 1)
    ni = np.bincount(row(common), minlength=n + 1)
    pts = np.arange(1, n + 1) if points is None else np.asarray(points, dtype=np.int64)
    if pts.size == 0:
        return float("nan")
    if pts.max() >= na.size:
        # points beyond every listed index still count (both sets empty)
        size = int(pts.max()) + 1
        na, nb, ni = (np.pad(v, (0, max(0, size - v.size))) for v in (na, nb, ni))
    a, b, c = na[pts], nb[pts], ni[pts]
    union = a + b - c
    ratio = np.where((a == 0) & (b == 0), 1.0,
                     np.where((a == 0) | (b == 0), 0.0, c / np.maximum(union, 1)))
    return float(np.cumsum(ratio, dtype=np.float64)[-1] / len(pts))


def overlap_accuracy_sets(test: ResultSet, truth: ResultSet, points=None) -> float:
    """The reference loop itself (one set per point), kept to pin the
    vectorised form above (tests/test_host.py)."""
    if test.n != truth.n:
        raise ArgumentError(f"result sets cover different datasets: n={test.n} vs n={truth.n}")
    a = _neighbor_sets(test)
    b = _neighbor_sets(truth)
    pts = range(1, test.n + 1) if points is None else [int(p) for p in points]
    total = 0.0
    for p in pts:
        na, nb = a.get(p), b.get(p)
        if not na and not nb:
            total += 1.0
            continue
        if na is None or nb is None:
            continue
        total += len(na & nb) / len(na | nb)
    return total / len(pts)


@dataclass
class ErrorStats:
    matched_pairs: int
    defined: bool
    err_mean: float
    err_std: float
    histogram: np.ndarray
    bin_edges: np.ndarray


def _pair_keys(i, j) -> np.ndarray:
    return (np.asarray(i).astype(np.uint64) << np.uint64(32)) | np.asarray(j).astype(np.uint64)


def distance_error_stats(test: ResultSet, truth: ResultSet, bins: int = DEFAULT_ERROR_BINS) -> ErrorStats:
    """Signed sqrt-distance error over matched pairs (analysis.py:186-219)."""
    if bins < 1:
        raise ArgumentError(f"bins must be >= 1, got {bins}")
    if test.n != truth.n:
        raise ArgumentError(f"result sets cover different datasets: n={test.n} vs n={truth.n}")
    _, ti, ui = np.intersect1d(_pair_keys(test.i, test.j), _pair_keys(truth.i, truth.j),
                               return_indices=True)
    if ti.size == 0:
        return ErrorStats(0, False, float("nan"), float("nan"), np.zeros(bins, np.int64),
                          np.linspace(0.0, 1.0, bins + 1))
    err = np.sqrt(test.dist_sq[ti].astype(np.float64)) - np.sqrt(truth.dist_sq[ui].astype(np.float64))
    hist, edges = np.histogram(err, bins=bins)
    return ErrorStats(int(ti.size), True, float(err.mean()), float(err.std()), hist, edges)


def pairwise_sqdist_fp64(values: np.ndarray, rows=None) -> np.ndarray:
    """FP64 direct-form squared distances, ascending k (oracle.py:26-40)."""
    x = np.asarray(values, dtype=np.float64)
    sel = x if rows is None else x[rows]
    acc = np.zeros((sel.shape[0], x.shape[0]), dtype=np.float64)
    for k in range(x.shape[1]):
        t = sel[:, k][:, None] - x[:, k][None, :]
        acc += t * t
    return acc


def brute_force_fp64_rows(values: np.ndarray, epsilon: float, rows) -> tuple:
    """FP64 truth for a row sample (brute_force_fp64, oracle.py:43-64,
    restricted to `rows`, 0-based): returns 1-based (i, j, d2)."""
    rows = np.asarray(rows)
    d2 = pairwise_sqdist_fp64(values, rows)
    keep = np.sqrt(d2) <= epsilon
    rr, cc = np.nonzero(keep)
    return (rows[rr] + 1).astype(np.uint32), (cc + 1).astype(np.uint32), d2[rr, cc]


@dataclass(frozen=True)
class CalibrationResult:
    epsilon: float
    estimated_selectivity: float
    iterations: int
    sample_size: int


def calibrate_epsilon(values: np.ndarray, target_s: float, tol: float = 0.05,
                      sample: int | None = None, seed: int = 0, max_iter: int = 40) -> CalibrationResult:
    """Bisection on an FP64 sample, same procedure and numbers as
    analysis.py:237-300 (accepts a Dataset or its values)."""
    values = getattr(values, "values", values)
    n = values.shape[0]
    if target_s <= 0:
        raise ArgumentError(f"target_s must be > 0, got {target_s}")
    if sample is None:
        sample = min(n, 1024)
    if not 2 <= sample <= n:
        raise ArgumentError(f"sample must be in [2, n={n}], got {sample}")
    if target_s > n - 1:
        raise CalibrationError(
            f"target selectivity {target_s} unreachable: at most n - 1 = {n - 1} neighbors exist")
    rng = np.random.default_rng(seed)
    idx = np.sort(rng.choice(n, size=sample, replace=False))
    m = int(sample)
    dist = np.sqrt(pairwise_sqdist_fp64(values[idx]))
    scale = (n - 1) / (m - 1)

    def estimate(eps: float) -> float:
        return scale * (int(np.count_nonzero(dist <= eps)) - m) / m

    band = tol * target_s
    lo, est_lo = 0.0, estimate(0.0)
    if abs(est_lo - target_s) <= band:
        return CalibrationResult(lo, est_lo, 0, m)
    if est_lo > target_s:
        raise CalibrationError(f"initial interval does not bracket target {target_s}: "
                               f"selectivity is already {est_lo:.4g} at epsilon 0")
    hi = float(dist.max())
    est_hi = estimate(hi)
    if est_hi < target_s - band:
        raise CalibrationError(f"initial interval does not bracket target {target_s}: "
                               f"achieved selectivity range is [{est_lo:.4g}, {est_hi:.4g}]")
    mid, est_mid = hi, est_hi
    for it in range(1, max_iter + 1):
        mid = 0.5 * (lo + hi)
        est_mid = estimate(mid)
        if abs(est_mid - target_s) <= band:
            return CalibrationResult(mid, est_mid, it, m)
        if est_mid < target_s:
            lo = mid
        else:
            hi = mid
    return CalibrationResult(mid, est_mid, max_iter, m)


@dataclass
class BandReport:
    """Parity of a test pair set against the reference pair set.

    Out-of-band mismatches are the contract violations (must be 0): pairs
    present on one side only whose REFERENCE distance lies outside
    |d2_ref - eps^2| <= band * eps^2."""

    ref_pairs: int
    test_pairs: int
    missing_in_band: int
    missing_out_of_band: int
    extra_in_band: int
    extra_out_of_band: int
    max_rel_dd2_matched: float    # max |d2_test - d2_ref| / eps^2 over matched pairs
    stricter_band_mismatches: int  # mismatches outside 0.1 * band

    @property
    def ok(self) -> bool:
        return self.missing_out_of_band == 0 and self.extra_out_of_band == 0


def band_compare(test_i, test_j, test_d, ref_i, ref_j, ref_d, eps_sq: float,
                 ref_d2_of_extra, band: float = 1e-3) -> BandReport:
    """Classify disagreements.  ``ref_d2_of_extra(i, j)`` returns the
    reference dist_sq of pairs the test found but the reference did not
    (they are absent from the reference lists)."""
    tk = _pair_keys(test_i, test_j)
    rk = _pair_keys(ref_i, ref_j)
    common, ti, ri = np.intersect1d(tk, rk, assume_unique=True, return_indices=True)
    eps_sq = float(eps_sq)
    scale = eps_sq if eps_sq > 0 else 1.0
    miss = np.setdiff1d(np.arange(len(rk)), ri, assume_unique=True)
    extra = np.setdiff1d(np.arange(len(tk)), ti, assume_unique=True)
    miss_d = np.asarray(ref_d, np.float64)[miss]
    if extra.size:
        extra_d = np.asarray(ref_d2_of_extra(np.asarray(test_i)[extra], np.asarray(test_j)[extra]),
                             np.float64)
    else:
        extra_d = np.zeros(0)
    lim = band * eps_sq
    rel = np.abs(np.asarray(test_d, np.float64)[ti] - np.asarray(ref_d, np.float64)[ri]) / scale
    return BandReport(
        ref_pairs=int(len(rk)), test_pairs=int(len(tk)),
        missing_in_band=int(np.count_nonzero(np.abs(miss_d - eps_sq) <= lim)),
        missing_out_of_band=int(np.count_nonzero(np.abs(miss_d - eps_sq) > lim)),
        extra_in_band=int(np.count_nonzero(np.abs(extra_d - eps_sq) <= lim)),
        extra_out_of_band=int(np.count_nonzero(np.abs(extra_d - eps_sq) > lim)),
        max_rel_dd2_matched=float(rel.max()) if rel.size else 0.0,
        stricter_band_mismatches=int(np.count_nonzero(np.abs(miss_d - eps_sq) > 0.1 * lim)
                                     + np.count_nonzero(np.abs(extra_d - eps_sq) > 0.1 * lim)),
    )
