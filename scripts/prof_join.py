"""Run only the join kernel on a workload (for ncu / quick timing).
usage: python scripts/prof_join.py C2 [reps] [exact]"""
import sys, os, time, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2508_21230_b200 as F
from paper_2508_21230_b200 import engine, _lib
from bench import WORKLOADS, SEED
wl = sys.argv[1] if len(sys.argv) > 1 else "C2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
exact = len(sys.argv) > 3 and sys.argv[3] == "exact"
name, n, d, eps = WORKLOADS[wl]
hd = F.to_half(F.generate_synthetic(n, d, seed=SEED))
dd = engine.upload(hd, 0)
es = float(np.float32(np.float32(eps) ** 2))
for r in range(reps):
    res = engine.join_device(dd, es, exact=exact, sort=(r == reps - 1))
    flops = 2.0 * n * n * d
    print(f"{wl} rep {r}: count {res.count} kernel {res.kernel_ms:.3f} ms "
          f"{flops / res.kernel_ms / 1e9:.1f} TFLOPS sort {res.sort_ms:.3f} ms", flush=True)
