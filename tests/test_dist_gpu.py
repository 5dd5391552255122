"""The product's one-process-per-GPU shard path (north star (4)),
run as two processes on one B200 (the driver's boxes have one GPU; gloo is
the process-group backend because NCCL refuses two ranks on one device).

Each rank calls the public ``self_join(hd, eps, shard=(rank, 2))`` -- the
tcgen05 kernels on its own 128-row-block range against every column -- and
``dist.gather_shards`` brings the rank-ordered parts to rank 0, whose
concatenation must equal the single-process ResultSet bit for bit.  The
second test runs ``bench.py --gpus 2`` under torchrun (gloo, both ranks on
cuda:0) so the N>1 bench line -- max-over-ranks timing, summed counts,
rank-0 cpu_baseline -- is exercised end to end.
"""

import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, d, eps, outq):
    import torch
    import torch.distributed as dist

    sys.path.insert(0, ROOT)
    import paper_2508_21230_b200 as F
    from paper_2508_21230_b200 import dist as fdist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        hd = F.to_half(F.generate_synthetic(n, d, seed=21))
        st = F.EngineStats()
        rs = F.self_join(hd, eps, stats_out=st, shard=(rank, world))
        rows = fdist.shard_rows(hd.n_padded, rank, world)
        assert rs.i.size == 0 or (rs.i.min() > rows[0] and rs.i.max() <= rows[1])
        merged = fdist.gather_shards((rs.i, rs.j, rs.dist_sq))
        total = fdist.reduce_sum(len(rs))
        t_max = fdist.reduce_max(st.kernel_wall_seconds)
        if rank == 0:
            outq.put((merged, total, t_max, st.kernel_wall_seconds))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_two_process_shards_equal_single_process():
    import torch.multiprocessing as mp

    import paper_2508_21230_b200 as F

    n, d, eps = 20000, 128, 3.8
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n, d, eps, q)) for r in range(2)]
    for p in procs:
        p.start()
    (mi, mj, md), total, t_max, t0 = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    ref = F.self_join(F.to_half(F.generate_synthetic(n, d, seed=21)), eps)
    assert len(ref) > n and total == len(ref)
    assert np.array_equal(mi, ref.i) and np.array_equal(mj, ref.j)
    assert np.array_equal(md.view(np.uint32), ref.dist_sq.view(np.uint32))
    assert t_max >= t0 > 0


@pytest.mark.gpu
def test_bench_two_ranks_under_torchrun():
    env = dict(os.environ, FASTED_BENCH_DIST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.join(ROOT, "bench.py"), "--gpus", "2", "--workload", "C1", "--steps", "3",
           "--warmup", "3", "--e2e-steps", "1", "--no-accuracy", "--ref-seconds", "1"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["value"] > 0 and line["e2e"]["value"] > 0
    assert line["pairs"] > 16384
    assert line["cpu_baseline"]["value"] > 0 and line["cpu_baseline"]["cores"] >= 1
    assert line["configs"] is None
