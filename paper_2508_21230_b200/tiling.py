"""Epsilon self-join drop-in (mirrors /root/reference/pkg/src/mpjoin/tiling.py).

``self_join`` keeps the reference signature, validation, epsilon handling
and ``ResultSet`` contract (1-based uint32 (i, j), FP32 dist_sq, canonical
(i, j) order, self pairs present) but the sweep runs on B200s:

* ``mode="tc"`` (default): the fused tcgen05 kernel.  Pairs match the
  reference exactly except possibly for pairs whose reference distance lies
  within the stated relative band (1e-3) of eps^2 -- the tensor core sums the
  FP32 products of a_ij in a different order than the reference's
  sequential round-toward-zero chain.
* ``mode="exact"``: the CUDA-core FFMA.RZ kernel, bit-identical to the
  reference (same pairs, same dist_sq bits).

``TileConfig`` is accepted and validated exactly as the reference does
(tiling.py:57-75, 174-184) so callers keep working; the GPU tile shape is a
compile-time property of the kernels (128x256 CTA tiles, 4-stage TMA ring).
``cfg.workers`` has no effect; ``devices=`` selects the GPUs instead.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np

from . import engine
from .dataset import HalfDataset
from .errors import ArgumentError, ConfigError

__all__ = [
    "TileConfig",
    "TileCoord",
    "ResultSet",
    "EngineStats",
    "rasterize_tiles",
    "compute_block_tile",
    "make_result_set",
    "self_join",
]

GPU_TILE_M, GPU_TILE_N = 128, 256


@dataclass
class TileConfig:
    """Tiling parameters, validated like the reference (tiling.py:44-75)."""

    block_side: int = 128
    block_kslice: int = 64
    warp_side: int = 64
    warp_kslice: int = 16
    dispatch_square: int = 8
    prefetch_depth: int = 2
    workers: int = 1
    raster_order: bool = True

    def validate(self) -> None:
        if self.warp_kslice != 16:
            raise ConfigError(f"warp_kslice must be 16, got {self.warp_kslice}")
        if self.warp_side < 16 or self.warp_side % 16 != 0:
            raise ConfigError(f"warp_side {self.warp_side} must be a positive multiple of 16")
        if self.block_side % self.warp_side != 0:
            raise ConfigError(
                f"block_side {self.block_side} not divisible by warp_side {self.warp_side}")
        if self.block_kslice < self.warp_kslice or self.block_kslice % self.warp_kslice != 0:
            raise ConfigError(
                f"block_kslice {self.block_kslice} not a multiple of warp_kslice {self.warp_kslice}")
        if self.dispatch_square < 1:
            raise ConfigError(f"dispatch_square must be >= 1, got {self.dispatch_square}")
        if self.prefetch_depth not in (1, 2):
            raise ConfigError(f"prefetch_depth must be 1 or 2, got {self.prefetch_depth}")
        if self.workers < 1:
            raise ConfigError(f"workers must be >= 1, got {self.workers}")


@dataclass(frozen=True)
class TileCoord:
    row_block: int
    col_block: int


@dataclass
class ResultSet:
    """Pairs (i, j, dist_sq) with dist <= epsilon, sorted by (i, j)
    (tiling.py:84-113)."""

    i: np.ndarray
    j: np.ndarray
    dist_sq: np.ndarray
    n: int
    epsilon: float

    def __len__(self) -> int:
        return int(self.i.shape[0])

    def index_pairs(self) -> set:
        return set(zip(self.i.tolist(), self.j.tolist()))

    def as_tuples(self):
        return list(zip(self.i.tolist(), self.j.tolist(), self.dist_sq.tolist()))

    def same_pairs(self, other: "ResultSet") -> bool:
        return (len(self) == len(other) and np.array_equal(self.i, other.i)
                and np.array_equal(self.j, other.j))


def make_result_set(i, j, dist_sq, n: int, epsilon: float) -> ResultSet:
    """Canonicalise host pair arrays by (i, j) (tiling.py:116-122)."""
    i = np.asarray(i, dtype=np.uint32)
    j = np.asarray(j, dtype=np.uint32)
    dist_sq = np.asarray(dist_sq)
    order = np.lexsort((j, i))
    return ResultSet(i[order], j[order], dist_sq[order], n=int(n), epsilon=float(epsilon))


@dataclass
class EngineStats:
    """Phase timings and work counters (tiling.py:125-151), filled from the
    GPU run: tiles/staged/reuse counters describe the 128x256 CTA tiles the
    tcgen05 kernel actually walks; kernel_wall_seconds is the CUDA-event time
    of the join kernel (max over devices)."""

    tiles: int = 0
    block_iterations: int = 0
    staged_elements: int = 0
    element_reads: int = 0
    fma_ops: int = 0
    stage_seconds: float = 0.0
    kernel_cpu_seconds: float = 0.0
    kernel_wall_seconds: float = 0.0
    merge_seconds: float = 0.0
    wall_seconds: float = 0.0
    per_device: list = field(default_factory=list)   # engine per-GPU report (chunks, host ms)

    @property
    def reuse_per_staged_element(self) -> float:
        return self.element_reads / self.staged_elements if self.staged_elements else 0.0

    def add(self, other: "EngineStats") -> None:
        self.tiles += other.tiles
        self.block_iterations += other.block_iterations
        self.staged_elements += other.staged_elements
        self.element_reads += other.element_reads
        self.fma_ops += other.fma_ops
        self.stage_seconds += other.stage_seconds
        self.kernel_cpu_seconds += other.kernel_cpu_seconds


def rasterize_tiles(grid_rows: int, grid_cols: int, square: int) -> list:
    """All tile coordinates in square x square groups (tiling.py:154-171)."""
    if grid_rows < 1 or grid_cols < 1:
        raise ArgumentError("grid dimensions must be >= 1")
    if square < 1:
        raise ArgumentError("square must be >= 1")
    coords = []
    for gr in range(0, grid_rows, square):
        for gc in range(0, grid_cols, square):
            for r in range(gr, min(gr + square, grid_rows)):
                for c in range(gc, min(gc + square, grid_cols)):
                    coords.append(TileCoord(r, c))
    return coords


def _check_engine_inputs(hd: HalfDataset, cfg: TileConfig) -> None:
    cfg.validate()
    if hd.n_padded % cfg.block_side != 0:
        raise ConfigError(
            f"n_padded {hd.n_padded} not a multiple of block_side {cfg.block_side}; "
            f"re-pad the dataset for this configuration")
    if hd.d_padded % cfg.warp_kslice != 0:
        raise ConfigError(f"d_padded {hd.d_padded} not a multiple of warp_kslice {cfg.warp_kslice}")


FLT_MAX = np.float32(np.finfo(np.float32).max)


def _eps_sq(epsilon) -> np.float32:
    """eps32 = f32(eps); eps_sq = f32(eps32 * eps32) (tiling.py:304-305).

    Where the reference's square overflows to inf (eps above ~1.8e19, or an
    eps that is itself beyond FP32 range) every finite dist_sq is <= inf, so
    it returns all n^2 pairs; clamping to FLT_MAX selects the same set and
    keeps the C ABI's finite-eps_sq contract."""
    with np.errstate(over="ignore"):
        eps32 = np.float32(epsilon)
        es = np.float32(eps32 * eps32)
    return es if es <= FLT_MAX else FLT_MAX


def _default_devices():
    import torch

    return [torch.cuda.current_device()] if torch.cuda.is_available() else [0]


def compute_block_tile(hd: HalfDataset, coord: TileCoord, eps_sq, cfg: TileConfig,
                       stats: EngineStats | None = None, device: int | None = None):
    """All within-threshold pairs of one block tile (tiling.py:199-285), on
    the GPU with the bit-exact kernel.  Returns (i, j, dist_sq) in the
    reference's row-major tile order."""
    _check_engine_inputs(hd, cfg)
    side = cfg.block_side
    grid = hd.n_padded // side
    if not (0 <= coord.row_block < grid and 0 <= coord.col_block < grid):
        raise ArgumentError(f"tile {coord} outside {grid}x{grid} grid")
    eps_sq = np.float32(eps_sq)
    if eps_sq < 0:
        raise ArgumentError("eps_sq must be >= 0")
    if stats is None:
        stats = EngineStats()
    dev = _default_devices()[0] if device is None else device
    dd = engine.upload(hd, dev)
    r0, c0 = coord.row_block * side, coord.col_block * side
    # kernel ranges are 128-aligned; cover the tile and trim afterwards
    rr = (r0 // 128 * 128, min(-(-(r0 + side) // 128) * 128, dd.n_dev))
    cc = (c0 // 128 * 128, min(-(-(c0 + side) // 128) * 128, dd.n_dev))
    res = engine.join_device(dd, float(eps_sq), rows=rr, cols=cc, exact=True)
    i, j, d = engine.to_host(res)
    keep = (i > r0) & (i <= r0 + side) & (j > c0) & (j <= c0 + side)
    stats.tiles += 1
    stats.fma_ops += side * side * hd.d_padded
    stats.kernel_wall_seconds += res.kernel_ms / 1e3
    return i[keep], j[keep], d[keep]


def self_join(hd: HalfDataset, epsilon: float, cfg: TileConfig | None = None,
              stats_out: EngineStats | None = None, *, mode: str = "tc",
              devices=None, shard=None, symmetric: bool = False) -> ResultSet:
    """Full epsilon self-join: every ordered pair with distance <= epsilon
    (tiling.py:288-359), on one or more B200s.

    mode "tc" is the tcgen05 product path; "exact" reproduces the reference
    bit for bit.  devices: list of CUDA device indices (row-block sharded,
    no collectives); default the current device.  shard=(rank, world): one
    process per GPU -- this call returns only the pairs whose i lies in the
    rank's contiguous row-block range; concatenating ranks in order gives
    the full, sorted ResultSet.  symmetric=True (tcgen05, one device, no
    shard): compute only the tiles on or above the diagonal and mirror each
    pair -- half the MMA work; every (i, j) then carries exactly the dist_sq
    of (j, i), so the result is exactly symmetric.
    """
    if cfg is None:
        cfg = TileConfig()
    _check_engine_inputs(hd, cfg)
    if not np.isfinite(epsilon) or epsilon < 0:
        raise ArgumentError(f"epsilon must be finite and >= 0, got {epsilon}")
    if mode not in ("tc", "exact"):
        raise ArgumentError(f"mode must be 'tc' or 'exact', got {mode!r}")
    eps_sq = _eps_sq(epsilon)
    if devices is None:
        devices = _default_devices()
    if symmetric and (mode != "tc" or len(list(devices)) != 1 or shard is not None):
        raise ArgumentError("symmetric=True needs mode 'tc' on a single device without shard")
    row_range = None
    if shard is not None:
        rank, world = shard
        if not (0 <= rank < world):
            raise ArgumentError(f"shard {shard} invalid")
        n_dev = -(-hd.n_padded // 128) * 128
        row_range = engine.partition_rows(n_dev, world)[rank]
    t0 = time.perf_counter()
    i, j, d, rep = engine.self_join_devices(hd, float(eps_sq), list(devices),
                                            exact=(mode == "exact"), row_range=row_range,
                                            symmetric=symmetric)
    rs = ResultSet(i, j, d, n=int(hd.n_logical), epsilon=float(epsilon))
    if stats_out is not None:
        n_dev = -(-hd.n_padded // 128) * 128
        d_pad = hd.d_padded
        tiles = (n_dev // GPU_TILE_M) * (-(-n_dev // GPU_TILE_N))
        kblocks = -(-d_pad // 64)
        st = EngineStats(
            tiles=tiles,
            block_iterations=tiles * kblocks,
            staged_elements=tiles * (GPU_TILE_M + GPU_TILE_N) * d_pad,
            element_reads=tiles * 2 * GPU_TILE_M * GPU_TILE_N * d_pad,
            fma_ops=n_dev * n_dev * d_pad,
            stage_seconds=rep.stage_seconds,
        )
        stats_out.add(st)
        stats_out.kernel_wall_seconds = rep.kernel_seconds
        stats_out.merge_seconds = rep.merge_seconds
        stats_out.per_device = rep.per_device
        stats_out.wall_seconds = time.perf_counter() - t0
    return rs
