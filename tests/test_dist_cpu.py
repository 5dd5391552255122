"""World-size-2 gloo test of the sharded join's host logic (CPU only).

Each rank takes its row-block range (dist.shard_rows), runs the join of its
rows -- here the CPU oracle stands in for the device join, which is the
only GPU piece of the flow -- and the rank-ordered gather must equal the
single-process result exactly; timing/count reductions follow the bench's
max-over-ranks / sum rules.
"""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2508_21230_b200 import dist as fdist


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, x, eps, outq):
    from oracle import oracle as O

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        v16, norms, _ = O.to_half(x)
        r0, r1 = fdist.shard_rows(v16.shape[0], rank, world)
        i, j, d = O.join(v16, norms, x.shape[0], eps, rows=(r0, r1), threads=1)
        t_max = fdist.reduce_max(float(rank + 1))
        total = fdist.reduce_sum(len(i))
        merged = fdist.gather_shards((i, j, d))
        if rank == 0:
            outq.put((merged, t_max, total, (r0, r1)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_sharded_join_equals_single(world):
    from oracle import oracle as O

    rng = np.random.default_rng(3)
    x = rng.random((700, 24), dtype=np.float32)
    eps = 1.2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, x, eps, q)) for r in range(world)]
    for p in procs:
        p.start()
    merged, t_max, total, r = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    v16, norms, _ = O.to_half(x)
    i, j, d = O.join(v16, norms, x.shape[0], eps, threads=2)
    assert np.array_equal(merged[0], i) and np.array_equal(merged[1], j)
    assert np.array_equal(merged[2].view(np.uint32), d.view(np.uint32))
    assert t_max == float(world) and total == len(i)
    assert r == (0, 384)   # 6 row blocks of 128 over 2 ranks


def test_shard_rows_cover_and_balance():
    for n_pad in (128, 256, 1000064, 5000064):
        for world in (1, 2, 3, 4, 8):
            parts = [fdist.shard_rows(n_pad, r, world) for r in range(world)]
            assert parts[0][0] == 0 and parts[-1][1] == n_pad
            assert all(a[1] == b[0] for a, b in zip(parts, parts[1:]))
            sizes = [(b - a) // 128 for a, b in parts]
            assert max(sizes) - min(sizes) <= 1
            assert all(a % 128 == 0 for a, _ in parts)


def test_merge_rejects_unordered():
    with pytest.raises(AssertionError):
        fdist.merge_shards([(np.array([2], np.uint32), np.array([1], np.uint32), np.zeros(1)),
                            (np.array([1], np.uint32), np.array([1], np.uint32), np.zeros(1))])
