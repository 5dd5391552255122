"""Where the end-to-end self_join time goes at a workload (C4 default).
usage: python scripts/e2e_breakdown.py [C4]"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2508_21230_b200 as F  # noqa: E402
from bench import SEED, WORKLOADS  # noqa: E402
from paper_2508_21230_b200 import engine  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "C4"
name, n, d, eps = WORKLOADS[wl]
hd = F.to_half(F.generate_synthetic(n, d, seed=SEED), pin_host=True)
hd_host = F.HalfDataset(hd.n_logical, hd.d_logical, hd.values, hd.norms)
hd.device_cache.clear()
torch.cuda.empty_cache()
es = float(np.float32(np.float32(eps) ** 2))
for rep in range(3):
    T = {}
    t0 = time.perf_counter()
    dd = engine.upload(hd_host, 0)
    torch.cuda.synchronize()
    T["h2d"] = time.perf_counter() - t0
    t1 = time.perf_counter()
    res = engine.join_device(dd, es)
    T["join_device(total)"] = time.perf_counter() - t1
    T["  kernel(events)"] = res.kernel_ms / 1e3
    T["  sort(events)"] = res.sort_ms / 1e3
    t2 = time.perf_counter()
    out = engine.to_host(res)
    T["d2h(to_host)"] = time.perf_counter() - t2
    t3 = time.perf_counter()
    cat = [np.concatenate([x]) for x in out]
    T["np.concatenate"] = time.perf_counter() - t3
    del dd, res, out, cat
    torch.cuda.empty_cache()
    t4 = time.perf_counter()
    rs = F.self_join(hd_host, eps)
    T["self_join(public API)"] = time.perf_counter() - t4
    del rs
    print(f"rep {rep}: " + ", ".join(f"{k}={v * 1e3:.1f}ms" for k, v in T.items()), flush=True)
