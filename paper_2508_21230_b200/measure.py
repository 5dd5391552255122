"""Measurement helpers shared by `bench.py` and the `bench` CLI sweep.

* ``ClockSampler`` -- nvidia-smi SM clock + throttle reasons sampled during a
  timed region (B200_PROFILING.md's clocks line).
* ``timed_launches`` -- per-launch CUDA-event times on the launching stream.
* ``tensor_roofline`` -- achieved distance TFLOPS against the measured
  tensor peaks (MEASURED_PEAKS.json), burst for short launches, sustained
  for launches that run long enough to hit the power cap.
* ``time_join`` -- device time of the product join kernel alone
  (``fasted_join`` over a row range x all columns, records written), the
  kernel-only figure the reference's ``cmd_bench`` reports as
  ``kernel_seconds`` (cli.py:384-392).

None of this is on the join's data path.
"""

from __future__ import annotations

import json
import os
import statistics
import subprocess
import threading

__all__ = ["ClockSampler", "load_peaks", "timed_launches", "tensor_roofline", "time_join",
           "LONG_LAUNCH_MS", "SM_COUNT", "FLOP_PER_CLK_SM"]

LONG_LAUNCH_MS = 100.0   # launches longer than this are rated against the sustained peak
SM_COUNT = 148
FLOP_PER_CLK_SM = 8192   # dense FP16 tcgen05 rate per SM per clock
_ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def load_peaks(path: str | None = None):
    """(bf16 burst TFLOPS, bf16 sustained TFLOPS, HBM GB/s, source) from the
    driver-written MEASURED_PEAKS.json, else B200_PROFILING.md's fallback."""
    try:
        with open(path or os.path.join(_ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return (float(p["bf16_tflops"]), float(p.get("bf16_tflops_sustained", 0) or 0),
                float(p.get("hbm_gbs", 0) or 6540.5), "measured")
    except Exception:
        return 1590.0, 1400.0, 6540.5, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md)."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int, period_ms: int = 200):
        self.device = device
        self.period_ms = period_ms
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", str(self.period_ms)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx),
                "reasons": sorted(reasons), "samples": len(sm)}


def timed_launches(stream, fn, reps):
    """Per-launch CUDA-event times (ms) of `reps` back-to-back calls of `fn`
    on `stream` (the stream the kernels are launched on)."""
    import torch

    ev = [torch.cuda.Event(enable_timing=True) for _ in range(reps + 1)]
    ev[0].record(stream)
    for r in range(reps):
        fn()
        ev[r + 1].record(stream)
    ev[-1].synchronize()
    return [ev[r].elapsed_time(ev[r + 1]) for r in range(reps)]


def tensor_roofline(flops, launch_ms, clocks, peaks):
    """Tensor-pipe roofline of one launch doing `flops` algorithmic FLOP."""
    peak_burst, peak_sus, _, src = peaks
    long = launch_ms > LONG_LAUNCH_MS and peak_sus
    peak = peak_sus if long else peak_burst
    achieved = flops / (launch_ms / 1e3) / 1e12
    out = {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
           "frac": achieved / peak,
           "peak_source": f"{src} " + ("bf16_tflops_sustained (launch > 100 ms)" if long
                                       else "bf16_tflops burst (launch <= 100 ms)")}
    mhz = clocks.get("sm_mhz") if clocks else None
    if mhz:
        at_clock = FLOP_PER_CLK_SM * SM_COUNT * mhz * 1e6 / 1e12
        out["frac_of_tensor_rate_at_median_clock"] = achieved / at_clock
    return out


def time_join(dd, eps_sq: float, reps: int, warmup: int = 1, rows=None, clocks: bool = True):
    """Device time of the product join kernel(s) over `rows` x all columns
    of the resident `dd` (engine.DeviceData), records written into a buffer
    sized from an exact count pass, so the timed launches do exactly what
    ``self_join`` does minus the sort and the copies.

    Returns dict(launch_ms=[...], pairs=int, kernel=str, flags=int,
    clocks={...} or None)."""
    import torch

    from . import _lib, engine

    L = _lib.load()
    device = dd.device
    rows = rows or (0, dd.n_dev)
    cols = (0, dd.n_dev)
    stream = torch.cuda.current_stream(device)
    sp = stream.cuda_stream
    cnt = torch.zeros(2, dtype=torch.int64, device=f"cuda:{device}")
    engine.join_raw(dd, eps_sq, _lib.JOIN_COUNT, rows, cols, None, 0, cnt, sp)
    pairs = engine.read_counts(cnt, stream)[0]
    cap = pairs + engine.max_holes(device)
    flags = _lib.JOIN_TC | engine.form_hints(pairs, rows, cols)
    rec = torch.empty((max(cap, 1), 4), dtype=torch.int32, device=f"cuda:{device}")

    def step():
        engine.join_raw(dd, eps_sq, flags, rows, cols, rec, cap, cnt, sp)

    for _ in range(warmup):
        step()
    torch.cuda.synchronize(device)
    if clocks:
        with ClockSampler(device, period_ms=50) as clk:
            ms = timed_launches(stream, step, reps)
        clk_summary = clk.summary()
    else:
        ms = timed_launches(stream, step, reps)
        clk_summary = None
    got = engine.read_counts(cnt, stream)[0]
    if got != pairs:
        raise AssertionError(f"join count changed between launches: {got} vs {pairs}")
    kernel = L.fasted_join_kernel_name(dd.d_pad, rows[1] - rows[0], dd.n_dev, flags).decode()
    del rec
    return {"launch_ms": ms, "pairs": pairs, "kernel": kernel, "flags": flags,
            "clocks": clk_summary}
