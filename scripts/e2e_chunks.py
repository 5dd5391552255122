"""C4 end to end through self_join (pinned host dataset, H2D + D2H inside) for several
pipeline chunk counts (engine.PIPELINE_CHUNKS), alternating: wall seconds per call."""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2508_21230_b200 as F  # noqa: E402
from bench import SEED, WORKLOADS  # noqa: E402
from paper_2508_21230_b200 import engine  # noqa: E402

name, n, d, eps = WORKLOADS["C4"]
hd = F.to_half(F.generate_synthetic(n, d, seed=SEED), pin_host=True)
hd_host = F.HalfDataset(hd.n_logical, hd.d_logical, hd.values, hd.norms)
del hd
torch.cuda.empty_cache()
res = {k: [] for k in ((2, False), (2, True), (4, False), (4, True), (1, False))}
for r in range(4):
    for k in res:
        engine.PIPELINE_CHUNKS, engine.TAPER_CHUNKS = k
        st = F.EngineStats()
        t0 = time.perf_counter()
        rs = F.self_join(hd_host, eps, stats_out=st)
        ev = torch.cuda.Event()
        ev.record()
        ev.synchronize()
        dt = time.perf_counter() - t0
        if r:
            res[k].append((dt, st.kernel_wall_seconds, st.per_device[0]["chunks"]))
        del rs
for k, v in res.items():
    print(f"chunks/taper {k}: wall median {statistics.median(x[0] for x in v):.4f} s, kernels "
          f"{statistics.median(x[1] for x in v):.4f} s, chunks used {v[0][2]}", flush=True)
