"""Pair accuracy against FP64 at scale (the paper's Eq. 3 and Table 6 on
sampled rows).

The reference computes the FP64 truth with ``brute_force_fp64``
(oracle.py:43-64) on the CPU, which took 324 s at 16K x 128.  Here the truth
for a row sample comes from ``fasted_fp64_rows`` (csrc/fp64.cu), which uses
the same FP64 operation order on the original FP32 coordinates.  The
metrics are the reference's ``overlap_accuracy`` and
``distance_error_stats`` (analysis.py:127-219), restricted to the sampled
points.
"""

from __future__ import annotations

import numpy as np

from . import _lib, engine
from .analysis import distance_error_stats, overlap_accuracy
from .errors import ArgumentError
from .tiling import ResultSet

__all__ = ["fp64_truth_rows", "brute_force_fp64", "sample_row_blocks", "join_row_blocks", "accuracy_vs_fp64"]


def fp64_truth_rows(values: np.ndarray, rows, epsilon: float, device: int = 0,
                    chunk_rows: int = 8192):
    """FP64 truth pairs (1-based i, j, float64 dist_sq) for the 0-based
    query `rows` (None: every point), canonical order.  The FP32 matrix is
    uploaded once; queries run in chunks of `chunk_rows`, each chunk's
    record buffer grown to its exact count and rerun if it overflowed."""
    import torch

    if not np.isfinite(epsilon) or epsilon < 0:
        raise ArgumentError(f"epsilon must be finite and >= 0, got {epsilon}")
    _lib.require_device(device)
    L = _lib.load()
    vals = np.ascontiguousarray(values, dtype=np.float32)
    n, d = vals.shape
    rows = (np.arange(n, dtype=np.int64) if rows is None
            else np.ascontiguousarray(np.asarray(rows, dtype=np.int64)))
    dev = f"cuda:{device}"
    parts = []
    with torch.cuda.device(device):
        stream = torch.cuda.current_stream().cuda_stream
        x = torch.from_numpy(vals).to(dev)
        cnt = torch.zeros(1, dtype=torch.int64, device=dev)
        cap = max(min(len(rows), chunk_rows) * 512, 1024)
        rec = torch.empty((cap, 4), dtype=torch.int32, device=dev)
        for c0 in range(0, len(rows), chunk_rows):
            q = torch.from_numpy(rows[c0:c0 + chunk_rows]).to(dev)
            while True:
                _lib.check(L.fasted_fp64_rows(x.data_ptr(), n, d, q.data_ptr(), q.numel(),
                                              float(epsilon), rec.data_ptr(), cap,
                                              cnt.data_ptr(), stream), "fasted_fp64_rows")
                count = engine.read_counts(cnt)[0]
                if count <= cap:
                    break
                cap = count + count // 4
                rec = torch.empty((cap, 4), dtype=torch.int32, device=dev)
            parts.append(rec[:count].cpu().numpy())
    raw = np.concatenate(parts) if parts else np.empty((0, 4), np.int32)
    i = raw[:, 0].view(np.uint32).copy()
    j = raw[:, 1].view(np.uint32).copy()
    d2 = raw[:, 2:4].copy().view(np.float64).reshape(-1)
    order = np.lexsort((j, i))
    return i[order], j[order], d2[order]


def brute_force_fp64(ds, epsilon: float, device: int = 0, rows=None) -> ResultSet:
    """Drop-in for the reference's ``brute_force_fp64`` (oracle.py:43-64):
    every ordered pair (self-pairs included) with FP64 distance <= epsilon,
    direct subtract-square form in ascending k on the original FP32 values,
    threshold sqrt(d2) <= epsilon, float64 dist_sq, canonical order --
    computed by ``fasted_fp64_rows`` on the GPU (csrc/fp64.cu).  `rows`
    (0-based) restricts the query points (the truth of a row sample)."""
    values = getattr(ds, "values", ds)
    i, j, d2 = fp64_truth_rows(values, rows, epsilon, device)
    return ResultSet(i, j, d2, n=int(values.shape[0]), epsilon=float(epsilon))


def sample_row_blocks(n: int, blocks: int = 8, seed: int = 0, block: int = 128) -> np.ndarray:
    """0-based rows of `blocks` distinct random 128-row blocks (whole blocks,
    so a restricted join over them is a few kernel launches)."""
    nblk = -(-n // block)
    rng = np.random.default_rng(seed)
    picks = np.sort(rng.choice(nblk, size=min(blocks, nblk), replace=False))
    rows = np.concatenate([np.arange(b * block, min((b + 1) * block, n)) for b in picks])
    return rows.astype(np.int64)


def join_row_blocks(dd, epsilon: float, rows, exact: bool = False) -> ResultSet:
    """Mixed-precision join restricted to the 128-row blocks covering
    `rows` (all columns); `dd` is an engine.DeviceData."""
    from . import engine

    from .tiling import _eps_sq

    eps_sq = float(_eps_sq(epsilon))
    blocks = np.unique(np.asarray(rows, dtype=np.int64) // engine.BLOCK)
    parts = []
    for b in blocks:
        r0 = int(b) * engine.BLOCK
        res = engine.join_device(dd, eps_sq, rows=(r0, min(r0 + engine.BLOCK, dd.n_dev)),
                                 exact=exact)
        parts.append(engine.to_host(res))
    i = np.concatenate([p[0] for p in parts]) if parts else np.empty(0, np.uint32)
    j = np.concatenate([p[1] for p in parts]) if parts else np.empty(0, np.uint32)
    d = np.concatenate([p[2] for p in parts]) if parts else np.empty(0, np.float32)
    return ResultSet(i, j, d, n=int(dd.n_logical), epsilon=float(epsilon))


def _restrict(rs: ResultSet, rows: np.ndarray) -> ResultSet:
    keep = np.isin(rs.i.astype(np.int64) - 1, rows)
    return ResultSet(rs.i[keep], rs.j[keep], rs.dist_sq[keep], rs.n, rs.epsilon)


def accuracy_vs_fp64(values: np.ndarray, rs: ResultSet, epsilon: float, rows,
                     device: int = 0) -> dict:
    """Eq. 3 overlap and signed distance error of `rs` against the FP64
    truth, averaged over the sampled points `rows` (0-based)."""
    rows = np.asarray(rows, dtype=np.int64)
    ti, tj, td = fp64_truth_rows(values, rows, epsilon, device)
    truth = ResultSet(ti, tj, td, rs.n, epsilon)
    test = _restrict(rs, rows)
    ov = overlap_accuracy(test, truth, points=rows + 1)
    es = distance_error_stats(test, truth)
    return {"overlap": ov, "loss_pct": 100.0 * (1.0 - ov), "err_mean": es.err_mean,
            "err_std": es.err_std, "matched_pairs": es.matched_pairs,
            "truth_pairs": int(len(ti)), "test_pairs": int(len(test)),
            "sample_points": int(len(rows))}
