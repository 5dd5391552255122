"""In-process A/B of kernel env knobs (read by libfasted per launch): one
dataset, rounds of one launch per setting, alternating; prints per-setting
median / min / all ms and TFLOPS.
usage: python scripts/ab_env.py C3 ROUNDS "FASTED_RES_HIT=0" "FASTED_RES_HIT=2" ...
AB_SHARD=r/w joins only rank r's row shard (all columns); AB_EPS overrides epsilon."""
import os
import statistics
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2508_21230_b200 as F  # noqa: E402
from bench import SEED, WORKLOADS  # noqa: E402
from paper_2508_21230_b200 import _lib, engine  # noqa: E402
# env knobs and diagnostic flags exist only in the experiment build
_lib.LIB_PATH = os.path.abspath(os.environ.get("FASTED_LIB", _lib.EXP_LIB_PATH))

wl, rounds = sys.argv[1], int(sys.argv[2])
settings = sys.argv[3:]
name, n, d, eps = WORKLOADS[wl]
eps = float(os.environ.get("AB_EPS", eps))
hd = F.to_half(F.generate_synthetic(n, d, seed=SEED))
dd = engine.upload(hd, 0)
es = float(np.float32(np.float32(eps) ** 2))
rank, world = (int(x) for x in os.environ.get("AB_SHARD", "0/1").split("/"))
rows = tuple(engine.partition_rows(dd.n_dev, world)[rank])
first = engine.join_device(dd, es, rows=rows, sort=False)
cap = first.count + engine.hole_slack(0)
ref = first.count
del first
rec = torch.empty((cap, 4), dtype=torch.int32, device="cuda")
cnt = torch.zeros(2, dtype=torch.int64, device="cuda")
s = torch.cuda.current_stream()
nrows = rows[1] - rows[0]
flags = _lib.JOIN_TC | engine.form_hints(ref, rows, (0, dd.n_dev))
times = {k: [] for k in settings}


extra = {}
# every env key any setting touches is reset to its starting value before
# each setting applies its own (settings do not leak into each other)
_keys = {kv.split("=")[0] for st in settings for kv in st.split(",") if not kv.startswith("F=")}
_orig = {k: os.environ.get(k) for k in _keys}


def apply(setting):
    extra.clear()
    for k, v in _orig.items():
        if v is None:
            os.environ.pop(k, None)
        else:
            os.environ[k] = v
    for kv in setting.split(","):
        k, v = kv.split("=")
        if k == "F":          # extra fasted_join flag bits for this setting
            extra["F"] = int(v)
        else:
            os.environ[k] = v


for r in range(rounds + 1):
    for st in settings:
        apply(st)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        engine.join_raw(dd, es, flags | extra.get("F", 0), rows, (0, dd.n_dev), rec, cap, cnt,
                        s.cuda_stream)
        e1.record(s)
        e1.synchronize()
        # diagnostic flags (>= 256) invalidate results, except the hit-search /
        # hand-off A/B flags (RARE_LM, RARE_ROWS, HITPACK, GENERICQ)
        if extra.get("F", 0) & ~(131072 | 262144 | 33554432 | 67108864 | 134217728 | 268435456) < 256:
            assert int(cnt[0]) == ref, (st, int(cnt[0]), ref)
        if r:   # round 0 warms up every setting
            times[st].append(e0.elapsed_time(e1))
fl = 2.0 * min(nrows, n) * n * d
for st, t in times.items():
    print(f"{wl} {st:28s} median {statistics.median(t):8.2f} ms ({fl / statistics.median(t) / 1e9:7.1f} "
          f"TFLOPS)  min {min(t):8.2f}  all {[round(x, 1) for x in t]}", flush=True)
