"""One-process-per-GPU plumbing for the sharded join (north star (4)).

The join shards by contiguous 128-row blocks with no data exchange: every
rank holds the full FP16 dataset and emits the pairs of its own rows.  The
only cross-rank traffic is bookkeeping -- the max of the per-rank device
times (the contract's timing rule) and the sum of the pair counts -- and,
when a caller wants the whole ResultSet on one host, a rank-ordered gather
(rank order == row order, so the concatenation is already canonical).
"""

from __future__ import annotations

import numpy as np

from .engine import BLOCK, partition_rows


def shard_rows(n_padded: int, rank: int, world: int) -> tuple:
    """[row_begin, row_end) of this rank (128-aligned, imbalance <= 1 block)."""
    n_dev = -(-n_padded // BLOCK) * BLOCK
    return partition_rows(n_dev, world)[rank]


def _device(device):
    """Where a bookkeeping tensor must live for the process group's backend:
    NCCL reduces only CUDA tensors (the current device), gloo CPU ones."""
    import torch
    import torch.distributed as dist

    if device is not None:
        return device
    if dist.get_backend() == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def reduce_max(value: float, device=None) -> float:
    """Max over ranks (the contract's timing rule: the job time is the
    slowest rank's device time)."""
    import torch
    import torch.distributed as dist

    if not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=_device(device))
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def reduce_sum(value: int, device=None) -> int:
    """Sum over ranks (pair counts: bookkeeping, not the data path)."""
    import torch
    import torch.distributed as dist

    if not dist.is_initialized() or dist.get_world_size() == 1:
        return int(value)
    t = torch.tensor([int(value)], dtype=torch.int64, device=_device(device))
    dist.all_reduce(t)
    return int(t.item())


def barrier() -> None:
    """Process-group barrier (no-op without one) followed by a device sync
    when CUDA is in use -- the bracket around every timed region."""
    import torch
    import torch.distributed as dist

    if dist.is_initialized() and dist.get_world_size() > 1:
        if dist.get_backend() == "nccl":
            dist.barrier(device_ids=[torch.cuda.current_device()])
        else:
            dist.barrier()
    if torch.cuda.is_available() and torch.cuda.is_initialized():
        torch.cuda.synchronize()


def merge_shards(parts) -> tuple:
    """Concatenate per-rank (i, j, d) in rank order; checks canonical order."""
    i = np.concatenate([np.asarray(p[0], np.uint32) for p in parts]) if parts else np.empty(0, np.uint32)
    j = np.concatenate([np.asarray(p[1], np.uint32) for p in parts]) if parts else np.empty(0, np.uint32)
    d = np.concatenate([np.asarray(p[2], np.float32) for p in parts]) if parts else np.empty(0, np.float32)
    if i.size > 1:
        key = (i.astype(np.uint64) << np.uint64(32)) | j.astype(np.uint64)
        if not np.all(key[1:] > key[:-1]):
            raise AssertionError("shards are not in canonical (i, j) order")
    return i, j, d


def gather_shards(local, dst: int = 0):
    """Gather every rank's (i, j, d) to `dst` (host objects over the process
    group: gather_object pickles through the backend -- CPU tensors on gloo,
    the current CUDA device on NCCL); returns the merged arrays on dst, None
    elsewhere."""
    import torch.distributed as dist

    if not dist.is_initialized() or dist.get_world_size() == 1:
        return merge_shards([local])
    out = [None] * dist.get_world_size() if dist.get_rank() == dst else None
    dist.gather_object(local, out, dst=dst)
    return merge_shards(out) if dist.get_rank() == dst else None
