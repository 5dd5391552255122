"""Sweep kernel variants (env knobs read per launch) on one workload and
report ms/launch, TFLOPS, SM clock and power.
usage: python scripts/tune.py C4 reps "CG=2,G=8192" "CG=1,G=2048" ..."""
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


wl, reps = sys.argv[1], int(sys.argv[2])
configs = sys.argv[3:] or ["CG=2,G=8192"]
name, n, d, eps = WORKLOADS[wl]
hd = F.to_half(F.generate_synthetic(n, d, seed=SEED))
dd = engine.upload(hd, 0)
es = float(np.float32(np.float32(eps) ** 2))
first = engine.join_device(dd, es, sort=False)
cap = first.count + engine.hole_slack(0)
ref_count = first.count
del first
rec = torch.empty((cap, 4), dtype=torch.int32, device="cuda")
cnt = torch.zeros(2, dtype=torch.int64, device="cuda")
stream = torch.cuda.current_stream()
try:
    import pynvml
    pynvml.nvmlInit()
    _nv = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
    energy_mj = lambda: pynvml.nvmlDeviceGetTotalEnergyConsumption(_nv)
except Exception:
    energy_mj = lambda: float("nan")


def sampler(stop, out):
    p = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw",
                          "--format=csv,noheader,nounits", "-lms", "100"],
                         stdout=subprocess.PIPE, text=True)
    while not stop.is_set():
        ln = p.stdout.readline()
        if ln:
            out.append((time.perf_counter(), ln))
    p.terminate()


for cfg in configs:
    kv = dict(x.split("=") for x in cfg.split(","))
    os.environ["FASTED_CTA_GROUP"] = kv.get("CG", "0")
    if "G" in kv:
        os.environ["FASTED_GROUP_ROWS"] = kv["G"]
    else:
        os.environ.pop("FASTED_GROUP_ROWS", None)
    os.environ["FASTED_RESIDENT"] = kv.get("R", "1")
    if "SEG" in kv:
        os.environ["FASTED_SEG_TILES"] = kv["SEG"]
    else:
        os.environ.pop("FASTED_SEG_TILES", None)
    os.environ["FASTED_MC"] = kv.get("MC", "1")
    os.environ["FASTED_RES_EPI"] = kv.get("EPI", "16")
    os.environ["FASTED_STREAM_EPI"] = kv.get("SEPI", "16")
    os.environ["FASTED_MC_EPI"] = kv.get("MEPI", "16")
    os.environ["FASTED_TS"] = kv.get("TS", "0")
    os.environ["FASTED_DYN"] = kv.get("DYN", "1")
    # default: the kernel-form hints the engine would pass for this output
    flags = int(kv.get("F", str(engine.form_hints(ref_count, (0, dd.n_dev), (0, dd.n_dev)))))
    engine.join_raw(dd, es, flags, (0, dd.n_dev), (0, dd.n_dev), rec, cap, cnt, stream.cuda_stream)
    torch.cuda.synchronize()
    time.sleep(1.0)
    out, stop = [], threading.Event()
    th = threading.Thread(target=sampler, args=(stop, out))
    th.start()
    time.sleep(0.3)
    t0 = time.perf_counter()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    j0 = energy_mj()
    e0.record(stream)
    for _ in range(reps):
        engine.join_raw(dd, es, flags, (0, dd.n_dev), (0, dd.n_dev), rec, cap, cnt,
                        stream.cuda_stream)
    e1.record(stream)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    joules = (energy_mj() - j0) / 1e3 / reps
    stop.set()
    th.join()
    ms = e0.elapsed_time(e1) / reps
    sel = [ln for (t, ln) in out if t0 + 0.25 * (t1 - t0) <= t <= t1]
    clk = [float(s.split(",")[0]) for s in sel]
    pw = [float(s.split(",")[1]) for s in sel]
    c = int(cnt[0].item())
    print(f"{wl} {cfg:22s} {ms:9.2f} ms {2.0 * n * n * d / ms / 1e9:8.1f} TFLOPS "
          f"clk {statistics.median(clk) if clk else float('nan'):6.0f} MHz "
          f"power {statistics.median(pw) if pw else float('nan'):6.0f} W "
          f"{joules:7.1f} J/launch {joules / (2.0 * n * n * d) * 1e12:6.3f} pJ/flop count {c}"
          f"{'' if c == ref_count else ' (COUNT DIFFERS from CG=2 default: %d)' % ref_count}",
          flush=True)
