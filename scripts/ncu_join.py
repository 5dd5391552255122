"""One warm + one measured join launch on a row slice of a workload (for ncu).
usage: python scripts/ncu_join.py C3 [rows] [flags]
The per-tile work is uniform, so rows [0, R) x all columns profiles the same
kernel behaviour as the full join in a fraction of the time."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2508_21230_b200 as F  # noqa: E402
from bench import SEED, WORKLOADS  # noqa: E402
from paper_2508_21230_b200 import _lib, engine  # noqa: E402

if os.environ.get("FASTED_LIB"):   # e.g. the experiment build (env knobs, diagnostic flags)
    _lib.LIB_PATH = os.path.abspath(os.environ["FASTED_LIB"])

wl = sys.argv[1]
rows = int(sys.argv[2]) if len(sys.argv) > 2 else 148 * 256 * 2
flags = int(sys.argv[3]) if len(sys.argv) > 3 else 0
name, n, d, eps = WORKLOADS[wl]
if len(sys.argv) > 4:
    eps = float(sys.argv[4])
hd = F.to_half(F.generate_synthetic(n, d, seed=SEED))
dd = engine.upload(hd, 0)
es = float(np.float32(np.float32(eps) ** 2))
r = (0, min(rows, dd.n_dev))
# explicit capacity: no count-only sizing launches before the measured one
first = engine.join_device(dd, es, rows=r, sort=False, capacity=(r[1] - r[0]) * 8192)
cap = first.count + engine.hole_slack(0)
rec = torch.empty((cap, 4), dtype=torch.int32, device="cuda")
cnt = torch.zeros(2, dtype=torch.int64, device="cuda")
s = torch.cuda.current_stream()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(s)
engine.join_raw(dd, es, flags, r, (0, dd.n_dev), rec, cap, cnt, s.cuda_stream)
e1.record(s)
torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
print(f"{wl} rows {r} flags {flags}: {ms:.3f} ms, {2.0 * (r[1] - r[0]) * n * d / ms / 1e9:.1f} "
      f"TFLOPS (rows x n x d), count {int(cnt[0])}")
