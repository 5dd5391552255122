"""Per-launch time vs SM clock for one workload (are slow launches clock events?).
usage: python scripts/outliers.py C3 24"""
import os
import subprocess
import sys
import threading
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2508_21230_b200 as F  # noqa: E402
from bench import SEED, WORKLOADS  # noqa: E402
from paper_2508_21230_b200 import _lib, engine  # noqa: E402

wl, n_launch = sys.argv[1], int(sys.argv[2])
name, n, d, eps = WORKLOADS[wl]
hd = F.to_half(F.generate_synthetic(n, d, seed=SEED))
dd = engine.upload(hd, 0)
es = float(np.float32(np.float32(eps) ** 2))
first = engine.join_device(dd, es, sort=False)
cap, ref = first.count + engine.hole_slack(0), first.count
del first
rec = torch.empty((cap, 4), dtype=torch.int32, device="cuda")
cnt = torch.zeros(2, dtype=torch.int64, device="cuda")
s = torch.cuda.current_stream()
flags = _lib.JOIN_TC | engine.form_hints(ref, (0, dd.n_dev), (0, dd.n_dev))
samples = []
stop = threading.Event()


def sampler():
    p = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,temperature.gpu,"
                          "clocks_event_reasons.active", "--format=csv,noheader,nounits",
                          "-lms", "20"], stdout=subprocess.PIPE, text=True)
    while not stop.is_set():
        ln = p.stdout.readline()
        if ln:
            samples.append((time.perf_counter(), ln.strip()))
    p.terminate()


th = threading.Thread(target=sampler)
th.start()
time.sleep(0.5)
rows = []
for k in range(n_launch):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record(s)
    engine.join_raw(dd, es, flags, (0, dd.n_dev), (0, dd.n_dev), rec, cap, cnt, s.cuda_stream)
    e1.record(s)
    e1.synchronize()
    t1 = time.perf_counter()
    rows.append((e0.elapsed_time(e1), t0, t1))
stop.set()
th.join()
for ms, t0, t1 in rows:
    sel = [x for (t, x) in samples if t0 <= t <= t1]
    clk = [float(x.split(",")[0]) for x in sel]
    pw = [float(x.split(",")[1]) for x in sel]
    reasons = sorted(set(x.split(",")[3].strip() for x in sel))
    print(f"{ms:8.2f} ms  clk {np.median(clk) if clk else float('nan'):6.0f} MHz (min "
          f"{min(clk) if clk else float('nan'):5.0f})  power {np.median(pw) if pw else float('nan'):5.0f} W"
          f"  reasons {reasons}", flush=True)
