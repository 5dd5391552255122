"""End-to-end public-API run of one 8-GPU rank's C5 shard (5M x 384) at a
given selectivity: H2D, chunked join -> sort -> D2H pipeline, pinned host
result arrays.  usage: python scripts/c5_e2e.py [eps] [shard r/8]"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2508_21230_b200 as F  # noqa: E402
from bench import SEED  # noqa: E402

eps = float(sys.argv[1]) if len(sys.argv) > 1 else 7.1352369182727085
rank, world = (int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "0/8").split("/"))
N, D = 5_000_000, 384
hd = F.to_half(F.generate_synthetic(N, D, seed=SEED), pin_host=True)
hd_host = F.HalfDataset(hd.n_logical, hd.d_logical, hd.values, hd.norms)
hd.device_cache.clear()
torch.cuda.empty_cache()
for rep in range(2):
    st = F.EngineStats()
    t0 = time.perf_counter()
    rs = F.self_join(hd_host, eps, stats_out=st, shard=(rank, world))
    wall = time.perf_counter() - t0
    ok_sorted = bool(np.all((np.diff(rs.i.astype(np.int64)) > 0) |
                            ((np.diff(rs.i.astype(np.int64)) == 0) & (np.diff(rs.j.astype(np.int64)) > 0))))
    rows = min(N, (-(-N // 128) * 128) * (rank + 1) // world) - (-(-N // 128) * 128) * rank // world
    e = st.per_device[0]
    print(json.dumps({"rep": rep, "eps": eps, "pairs": len(rs), "wall_s": wall,
                      "kernel_s": st.kernel_wall_seconds, "h2d_s": st.stage_seconds,
                      "not_hidden_s": st.merge_seconds, "chunks": e["chunks"],
                      "reruns": e["reruns"], "sort_ms": e["sort_ms"],
                      "canonical_order": ok_sorted,
                      "shard_tflops": 2.0 * rows * N * D / wall / 1e12,
                      "pairs_per_s": len(rs) / wall, "host_ms": e.get("host_ms")}), flush=True)
    del rs
