"""FaSTED epsilon self-join benchmark (driver contract: one JSON line).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload C4] [--impl reference]

A step is one full pass of the hot path over the workload: the fused
tcgen05 join (libfasted.so: fasted_join) of this rank's row-block range
against every column, FP16 dataset and norms resident in HBM (1.92 GB at C4,
far larger than the 126 MB L2, so no flush is needed between steps).
`value` = whole-job distance TFLOPS, 2 n^2 d / (max over ranks of the
per-step device time).  `e2e` is the same metric through the public API
(paper_2508_21230_b200.self_join on a pinned host HalfDataset: H2D of the
FP16 matrix + norms, join, device sort, D2H of the sorted pair list).

--impl reference times the reference's CPU path (the C oracle restatement
of mpjoin's RZ join, oracle/fasted_oracle.c, all host threads) on a bounded
sample of the same workload.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "ε-self-join TFLOPS, % of FP16 TC peak at 1–8 B200; pair accuracy vs FP64"

# SURVEY.md section 8 configs (eps from the reference CLI calibrate, seed 12345)
WORKLOADS = {
    "C1": ("synthetic uniform 16K x 128 (oracle config)", 16384, 128, 3.973260466174982),
    "C2": ("CIFAR-shaped synthetic 60K x 512", 60000, 512, 8.48414709018062),
    "C3": ("SIFT-shaped synthetic 1M x 128, S~64", 1000000, 128, 3.685431479161428),
    "C4": ("GIST-shaped synthetic 1M x 960, S~64", 1000000, 960, 11.700486640655093),
    "C5": ("Tiny-shaped synthetic 5M x 384, S~1024", 5000000, 384, 7.1352369182727085),
}
SEED = 12345


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["bf16_tflops"]), float(p.get("bf16_tflops_sustained", 0) or 0), "measured"
    except Exception:
        return 1590.0, 1400.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md)."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
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


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def cpu_sample(n, d, eps, seconds_target=12.0, threads=None):
    """Oracle (reference restatement) TFLOPS on a bounded sample: one
    128-row block of the workload against a column range sized so the run
    takes ~seconds_target.  Returns (tflops, sample description, threads)."""
    from oracle import oracle as O
    from paper_2508_21230_b200.dataset import synthetic_rows

    threads = threads or len(os.sched_getaffinity(0))
    rows = 128 * max(1, threads // 2)
    rows = min(rows, n - n % 128 if n >= 128 else n)
    cols = min(n, 4096)
    # calibrate on a small slab, then size the measured sample
    x = synthetic_rows(n, d, SEED, 0, max(rows, cols))
    v16, norms, _ = O.to_half(x)
    t0 = time.perf_counter()
    O.join(v16, norms, x.shape[0], eps, rows=(0, rows), cols=(0, min(cols, 1024)),
           threads=threads, count_only=True)
    dt = max(time.perf_counter() - t0, 1e-3)
    rate = 2.0 * rows * min(cols, 1024) * d / dt
    want_cols = int(min(n, max(1024, seconds_target * rate / (2.0 * rows * d))))
    want_cols = -(-want_cols // 128) * 128
    want_cols = min(want_cols, -(-n // 128) * 128)
    if want_cols > x.shape[0]:
        x = synthetic_rows(n, d, SEED, 0, min(n, want_cols))
        v16, norms, _ = O.to_half(x)
    cols_eff = min(want_cols, v16.shape[0])
    t0 = time.perf_counter()
    O.join(v16, norms, x.shape[0], eps, rows=(0, rows), cols=(0, cols_eff), threads=threads,
           count_only=True)
    dt = time.perf_counter() - t0
    tflops = 2.0 * rows * cols_eff * d / dt / 1e12
    return tflops, f"rows 0..{rows} x cols 0..{cols_eff} of {n}x{d} ({dt:.1f} s)", threads


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    name, n, d, eps = WORKLOADS[args.workload]
    threads = len(os.sched_getaffinity(0))
    vals = []
    desc = ""
    for s in range(args.warmup + args.steps):
        tf, desc, threads = cpu_sample(n, d, eps, seconds_target=args.ref_seconds, threads=threads)
        if s >= args.warmup:
            vals.append(tf)
    v = statistics.mean(vals)
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "TFLOPS",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        # the full workload on the CPU, extrapolated from the sampled rate
        "ms_per_step": 2.0 * n * n * d / (v * 1e12) * 1e3, "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None, "dtype": "fp16 in / fp32 RZ accumulate", "data": "synthetic",
        "config": {"workload": f"{args.workload}: {name}", "n": n, "d": d, "epsilon": eps,
                   "seed": SEED},
        "cpu_baseline": {"value": v, "unit": "TFLOPS", "cores": threads, "kind": "port",
                         "sample": desc},
        "e2e": {"value": v, "unit": "TFLOPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="C4", choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="fasted", choices=["fasted", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--ref-seconds", type=float, default=12.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-accuracy", action="store_true")
    ap.add_argument("--no-symmetric", action="store_true")
    ap.add_argument("--accuracy-blocks", type=int, default=8)
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import paper_2508_21230_b200 as F
    from paper_2508_21230_b200 import _lib, engine

    rank, world, local = dist_env()
    if world > 1:
        torch.cuda.set_device(local)
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    device = torch.cuda.current_device()
    _lib.require_device(device)
    name, n, d, eps = WORKLOADS[args.workload]

    # ---- data: every rank holds the full FP16 dataset
    ds = F.generate_synthetic(n, d, seed=SEED)
    hd = F.to_half(ds, pin_host=True)          # GPU quantise; device copy cached
    if rank != 0 or args.no_accuracy:
        del ds
    n_dev = -(-hd.n_padded // 128) * 128
    rows = engine.partition_rows(n_dev, world)[rank]
    dd = engine.upload(hd, device)
    eps_sq = float(np.float32(np.float32(eps) * np.float32(eps)))
    stream = torch.cuda.current_stream()
    # size the record buffer once (exact count + per-warp chunk slack)
    first = engine.join_device(dd, eps_sq, rows=rows, sort=False)
    cap = first.count + engine.hole_slack(device)
    del first
    rec = torch.empty((max(cap, 1), 4), dtype=torch.int32, device=f"cuda:{device}")
    cnt = torch.zeros(2, dtype=torch.int64, device=f"cuda:{device}")

    nrows = max(rows[1] - rows[0], 1)
    # the product path's kernel-form hint (engine.stream_join sets it the same way)
    jflags = _lib.JOIN_TC | engine.form_hints(cap - engine.hole_slack(device), rows, (0, dd.n_dev))

    def step():
        engine.join_raw(dd, eps_sq, jflags, rows, (0, dd.n_dev), rec, cap, cnt,
                        stream.cuda_stream)

    def barrier():
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        step()
    barrier()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    with ClockSampler(device) as clk:
        barrier()
        ev[0].record(stream)
        for s in range(args.steps):
            step()
            ev[s + 1].record(stream)
        torch.cuda.synchronize()
        barrier()
    per_step = [ev[s].elapsed_time(ev[s + 1]) for s in range(args.steps)]
    ms_local = ev[0].elapsed_time(ev[-1]) / args.steps
    # opt-in symmetric schedule (upper tiles + mirrored records; world == 1):
    # same record set, half the MMA work -- reported beside the headline,
    # which stays the full n^2 computation of the reference and the paper
    sym = None
    if world == 1 and not args.no_symmetric:
        def sym_step():
            engine.join_raw(dd, eps_sq, jflags | _lib.JOIN_SYMMETRIC, rows,
                            (0, dd.n_dev), rec, cap, cnt, stream.cuda_stream)
        sym_step()
        barrier()
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record(stream)
        for _ in range(max(1, args.steps // 2)):
            sym_step()
        s1.record(stream)
        torch.cuda.synchronize()
        sym_ms = s0.elapsed_time(s1) / max(1, args.steps // 2)
        sym_pairs = int(cnt[0].item())
        sym = {"ms_per_step": sym_ms, "pairs": sym_pairs,
               "time_to_solution_speedup": (ms_local / sym_ms),
               # 256 x 256 tiles on or above the diagonal (both kernel forms tile so)
               "executed_tflops": (lambda R: R * (R + 1) / 2 * 2.0 * 256 * 256 * d)(
                   -(-dd.n_dev // 256)) / (sym_ms / 1e3) / 1e12,
               "note": "self_join(..., symmetric=True): tiles on/above the diagonal only, "
                       "mirrored records; the headline value is the full n^2 computation"}
    pairs_local = int(cnt[0].item())
    ms = ms_local
    pairs = pairs_local
    if world > 1:
        t = torch.tensor([ms_local], dtype=torch.float64, device=f"cuda:{device}")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
        c = torch.tensor([pairs_local], dtype=torch.int64, device=f"cuda:{device}")
        torch.distributed.all_reduce(c)   # counts summed (bookkeeping, not data path)
        pairs = int(c.item())
    flops = 2.0 * n * n * d
    value = flops / (ms / 1e3) / 1e12
    peak_burst, peak_sus, peak_src = load_peaks()
    # A join launch at C4 runs ~1.4 s back to back under the 1 kW cap: the
    # "kernel inside a long step" case, whose denominator is the sustained
    # cuBLAS figure (B200_PROFILING.md); the burst fraction is kept beside it.
    peak = peak_sus if peak_sus else peak_burst
    peak_kind = "bf16_tflops_sustained" if peak_sus else "bf16_tflops (burst)"
    kernel_name = _lib.load().fasted_join_kernel_name(dd.d_pad, rows[1] - rows[0], dd.n_dev,
                                                      jflags).decode()
    # roofline of the dominant kernel (the join): algorithmic flops per launch
    rows_logical = max(0, min(rows[1], n) - min(rows[0], n))
    flops_launch = 2.0 * rows_logical * n * d
    avg_launch_ms = statistics.mean(per_step)
    achieved = flops_launch / (avg_launch_ms / 1e3) / 1e12
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            prof = json.load(f)
        traffic = prof.get(args.workload, {}).get("dram_bytes_per_launch")
    except Exception:
        pass
    del rec
    torch.cuda.empty_cache()

    # ---- e2e through the public API with host buffers (H2D + D2H inside)
    hd_host = F.HalfDataset(hd.n_logical, hd.d_logical, hd.values, hd.norms)  # no device cache
    del dd
    hd.device_cache.clear()
    torch.cuda.empty_cache()
    e2e_times = []
    phases = []
    d2h = 0
    for s in range(args.e2e_steps + 1):
        barrier()
        st = F.EngineStats()
        t0 = time.perf_counter()
        rs = F.self_join(hd_host, eps, stats_out=st, shard=(rank, world))
        # self_join returns host arrays after waiting for its own streams; the
        # device-wide check polls (a blocking sync can return 10-1000 ms late
        # here, see engine._poll)
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream())
        while not ev.query():
            time.sleep(0.0002)
        dt = time.perf_counter() - t0
        if s > 0:
            phases.append({"h2d_s": st.stage_seconds, "join_kernels_s": st.kernel_wall_seconds,
                           "sort_d2h_not_hidden_s": st.merge_seconds, "wall_s": dt,
                           "engine": st.per_device})
        if world > 1:
            t = torch.tensor([dt], dtype=torch.float64, device=f"cuda:{device}")
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            dt = float(t.item())
        if s > 0:          # first call warms the pinned-host caching allocator
            e2e_times.append(dt)
        d2h = len(rs) * 12
        del rs
    e2e_s = statistics.median(e2e_times)
    h2d = hd.values.nbytes + hd.norms.nbytes

    # ---- pair accuracy vs FP64 (Eq. 3) on sampled whole row blocks: the
    # tcgen05 path and the reference arithmetic (exact kernel) side by side
    acc = None
    if rank == 0 and not args.no_accuracy:
        from paper_2508_21230_b200 import accuracy

        arows = accuracy.sample_row_blocks(n, blocks=args.accuracy_blocks, seed=0)
        dd_a = engine.upload(hd, device)
        acc = {"sample": f"{args.accuracy_blocks} random 128-row blocks ({len(arows)} points) "
                         "x all columns; FP64 truth = fasted_fp64_rows (oracle.py order)"}
        for label, exact in (("tcgen05", False), ("reference_arithmetic_exact_kernel", True)):
            part = accuracy.join_row_blocks(dd_a, eps, arows, exact=exact)
            acc[label] = accuracy.accuracy_vs_fp64(ds.values, part, eps, arows, device)
        del dd_a, ds
        torch.cuda.empty_cache()

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            tf, desc, threads = cpu_sample(n, d, eps, seconds_target=args.ref_seconds)
            cpu = {"value": tf, "unit": "TFLOPS", "cores": threads, "kind": "port",
                   "sample": desc + "; oracle/fasted_oracle.c (RZ join restated from mpjoin)"}
        except Exception as exc:   # reported, never silently replaced
            cpu = {"value": None, "unit": "TFLOPS", "cores": None, "kind": "port",
                   "sample": f"failed: {exc}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "TFLOPS", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "fp16 in / fp32 accumulate (tcgen05 kind::f16)",
            "data": "synthetic uniform [0,1), generate_synthetic seed 12345",
            "config": {
                "workload": f"{args.workload}: {name}", "n": n, "d": d, "epsilon": eps,
                "eps_sq": eps_sq, "pairs": pairs, "selectivity": (pairs - n) / n,
                "parallelism": f"row-block shard x{world} (no collective)",
                "l2": "inputs %.2f GB >> 126 MB L2; no flush" % (h2d / 1e9),
            },
            "pct_of_fp16_peak": {"measured_burst": value / peak_burst, "measured_sustained":
                                 (value / peak_sus if peak_sus else None),
                                 "nominal_2250": value / 2250.0},
            "pairs_per_s": pairs / (ms / 1e3),
            "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak,
                         "unit": "TFLOP/s", "frac": achieved / peak, "traffic": traffic,
                         "peak_source": f"{peak_src} {peak_kind} (MEASURED_PEAKS.json)",
                         "frac_of_burst": achieved / peak_burst,
                         "kernel": kernel_name,
                         "launch_includes": "Gram-diagonal pre-pass + augment-row prep "
                                            "(~1/7800 of the join) + the join",
                         "output_write_bound_ms": pairs_local * 12 / 6552e9 * 1e3},
            "e2e": {"value": flops / e2e_s / 1e12, "unit": "TFLOPS",
                    "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "seconds_per_step": e2e_s, "api": "paper_2508_21230_b200.self_join",
                    "phases_per_step": phases},
            "accuracy_vs_fp64": acc,
            "symmetric_schedule": sym,
            # per step: Gram-diagonal pre-pass, aug_prepare_kernel, the join
            "gpu_launches": 3 * args.steps,
            "clocks": clk.summary(),
            "cpu_baseline": cpu,
            "per_step_ms": per_step,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
