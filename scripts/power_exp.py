"""Attribute the join kernel's power: run variants (normal / no epilogue /
no MMA / count-only) back to back and record time, SM clock and power.
usage: python scripts/power_exp.py C4 [reps]"""
import os
import statistics
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
# env knobs and diagnostic flags exist only in the experiment build
_lib.LIB_PATH = os.path.abspath(os.environ.get("FASTED_LIB", _lib.EXP_LIB_PATH))

wl = sys.argv[1] if len(sys.argv) > 1 else "C4"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
name, n, d, eps = WORKLOADS[wl]
hd = F.to_half(F.generate_synthetic(n, d, seed=SEED))
dd = engine.upload(hd, 0)
es = float(np.float32(np.float32(eps) ** 2))
first = engine.join_device(dd, es, sort=False)
cap = first.count + engine.hole_slack(0)
del first
rec = torch.empty((cap, 4), dtype=torch.int32, device="cuda")
cnt = torch.zeros(2, dtype=torch.int64, device="cuda")
stream = torch.cuda.current_stream()


def sampler(stop, out):
    p = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw",
                          "--format=csv,noheader,nounits", "-lms", "100"],
                         stdout=subprocess.PIPE, text=True)
    while not stop.is_set():
        ln = p.stdout.readline()
        if ln:
            out.append((time.perf_counter(), ln))
    p.terminate()


variants = [("normal", 0), ("count-only", _lib.JOIN_COUNT), ("no-epilogue", 256),
            ("load-only", 1024), ("sign-only", 2048), ("no-mma", 512), ("normal-again", 0)]
if len(sys.argv) > 3:
    variants = [v for v in variants if v[0] in sys.argv[3].split(",")]
for label, flags in variants:
    time.sleep(1.0)
    out, stop = [], threading.Event()
    th = threading.Thread(target=sampler, args=(stop, out))
    th.start()
    time.sleep(0.3)
    t0 = time.perf_counter()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(reps):
        engine.join_raw(dd, es, flags, (0, dd.n_dev), (0, dd.n_dev), rec, cap, cnt,
                        stream.cuda_stream)
    e1.record(stream)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    stop.set()
    th.join()
    ms = e0.elapsed_time(e1) / reps
    span = t1 - t0
    sel = [ln for (t, ln) in out if t0 + 0.25 * span <= t <= t1]
    clk = [float(s.split(",")[0]) for s in sel]
    pw = [float(s.split(",")[1]) for s in sel]
    print(f"{wl} {label:13s} {ms:9.2f} ms/launch {2.0 * n * n * d / ms / 1e9:8.1f} TFLOPS "
          f"clk {statistics.median(clk) if clk else float('nan'):6.0f} MHz "
          f"power {statistics.median(pw) if pw else float('nan'):6.0f} W  "
          f"count {int(cnt[0].item())}", flush=True)
