"""GPU timeline of the public self_join pipeline at C4 (join/sort events)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2508_21230_b200 as F  # noqa: E402
from bench import SEED, WORKLOADS  # noqa: E402

name, n, d, eps = WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "C4"]
hd = F.to_half(F.generate_synthetic(n, d, seed=SEED), pin_host=True)
hd_host = F.HalfDataset(hd.n_logical, hd.d_logical, hd.values, hd.norms)
hd.device_cache.clear()
for rep in range(4):
    st = F.EngineStats()
    t0 = time.perf_counter()
    rs = F.self_join(hd_host, eps, stats_out=st)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    print(json.dumps({"rep": rep, "wall_s": wall, "kernel_s": st.kernel_wall_seconds,
                      "h2d_s": st.stage_seconds, "engine": st.per_device}), flush=True)
    del rs
