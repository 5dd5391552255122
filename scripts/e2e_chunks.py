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
_plan = engine.plan_row_chunks
_upload = engine.upload_segmented


def head_plan(rows, est, budget, min_chunks=1, frac=16):
    """a first chunk of ~1/frac of the rows (starts after 1/frac of the upload), then the plan"""
    r0, r1 = rows
    cut = r0 + max(1, (r1 - r0) // engine.BLOCK // frac) * engine.BLOCK
    return [(r0, cut)] + _plan((cut, r1), est, budget, min_chunks)


res = {k: [] for k in ((2, False, 0, 16), (2, False, 0, 8), (2, False, 0, 4), (2, False, 0, 32))}
for r in range(4):
    for k in res:
        engine.PIPELINE_CHUNKS, engine.TAPER_CHUNKS = k[0], k[1]
        engine.upload_segmented = (lambda hd, dev, _s=k[3], _f=_upload: _f(hd, dev, segments=_s))
        engine.plan_row_chunks = (lambda *a, f=k[2]: head_plan(*a, frac=f)) if k[2] else _plan
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
