"""C5 selectivity sweep: Tiny-shaped synthetic 5M x 384, epsilon from self-pairs
only (eps = 0) to S ~ 4096 -- the output-compaction-bound regime.

One B200 runs exactly the work of ONE rank of the 8-GPU job (row shard r/8 of
the row blocks x all 5M columns, the full FP16 dataset resident): the path has
no exchange step, so the 8-GPU job time is the max over ranks of this time.
Per epsilon it reports, as one JSON line:
  * the count-only join (sign test + counting, no records) and the full
    pair-writing join, each as CUDA-event time of the launches, TFLOPS of the
    shard (2 rows n d) and pairs/s;
  * the device sort of the records into canonical (i, j) order;
  * the output-write roofline: record bytes / measured HBM copy bandwidth.
usage: python scripts/c5_sweep.py [--shard 0/8] [--reps 2]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2508_21230_b200 as F  # noqa: E402
from bench import SEED, ClockSampler, load_peaks  # noqa: E402
from paper_2508_21230_b200 import _lib, engine  # noqa: E402
# env knobs and diagnostic flags exist only in the experiment build
_lib.LIB_PATH = os.path.abspath(os.environ.get("FASTED_LIB", _lib.EXP_LIB_PATH))


# eps per target selectivity (reference CLI calibrate, sample 4096)
SWEEP = [("S0 (self pairs only)", 0.0), ("S16", 6.896041752764515), ("S64", 6.97276473038035),
         ("S256", 7.049487707996186), ("S1024", 7.1352369182727085),
         ("S4096", 7.2300123612099165)]
N, D = 5_000_000, 384


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shard", default="0/8")
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--only", default="")
    ap.add_argument("--extra-flags", default="0",
                    help="comma list of diagnostic flag sets to A/B (each row runs once per set)")
    args = ap.parse_args()
    extras = [int(x) for x in args.extra_flags.split(",")]
    rank, world = (int(x) for x in args.shard.split("/"))
    t0 = time.time()
    hd = F.to_half(F.generate_synthetic(N, D, seed=SEED))
    dd = engine.upload(hd, 0)
    rows = engine.partition_rows(dd.n_dev, world)[rank]
    nrows = min(rows[1], N) - min(rows[0], N)
    print(f"# data ready in {time.time() - t0:.1f} s; rows {rows} of {dd.n_dev}", flush=True)
    L = _lib.load()
    stream = torch.cuda.current_stream()
    sp = stream.cuda_stream
    hbm = 6540.5
    try:
        with open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                               "MEASURED_PEAKS.json")) as f:
            hbm = float(json.load(f)["hbm_gbs"])
    except Exception:
        pass
    peak_burst, peak_sus, _, _ = load_peaks()
    cnt = torch.zeros(2, dtype=torch.int64, device="cuda")
    flops = 2.0 * nrows * N * D
    for (label, eps), extra in [(le, x) for le in SWEEP for x in extras]:
        if args.only and args.only not in label:
            continue
        es = float(np.float32(np.float32(eps) * np.float32(eps)))

        def timed(fn):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            fn()
            e1.record(stream)
            e1.synchronize()
            return e0.elapsed_time(e1)

        # untimed count (sizes the record buffer and picks the kernel-form hint)
        engine.join_raw(dd, es, _lib.JOIN_COUNT, rows, (0, dd.n_dev), None, 0, cnt, sp)
        pairs = int(cnt[0].item())
        cap = pairs + engine.max_holes(0)
        jflags = _lib.JOIN_TC | extra | engine.form_hints(pairs, rows, (0, dd.n_dev))
        count_ms = []
        with ClockSampler(0) as clk_c:
            for _ in range(args.reps):
                count_ms.append(timed(lambda: engine.join_raw(
                    dd, es, jflags | _lib.JOIN_COUNT, rows, (0, dd.n_dev), None, 0, cnt, sp)))
        rec = torch.empty((cap, 4), dtype=torch.int32, device="cuda")
        join_ms = []
        with ClockSampler(0) as clk_j:
            for _ in range(args.reps):
                join_ms.append(timed(lambda: engine.join_raw(
                    dd, es, jflags, rows, (0, dd.n_dev), rec, cap, cnt, sp)))
        slots = int(cnt[1].item()) * engine.RECORD_CHUNK
        assert int(cnt[0].item()) == pairs
        dev = "cuda"
        sout = (torch.empty(max(pairs, 1), dtype=torch.int32, device=dev),
                torch.empty(max(pairs, 1), dtype=torch.int32, device=dev),
                torch.empty(max(pairs, 1), dtype=torch.float32, device=dev))
        stmp = torch.empty(max(pairs, 1), dtype=torch.int64, device=dev)   # 8-byte (j, d) scratch
        sws = torch.empty(L.fasted_sort_workspace_bytes(rows[1] - rows[0], dd.n_dev),
                          dtype=torch.uint8, device=dev)
        sort = lambda: engine._sort_records(dd, rec, slots, pairs, rows, stream, out=sout,
                                            timed=False, tmp=stmp, ws=sws)
        sort()   # first call: attributes, caches
        sort_ms = timed(sort)
        del sout, stmp, sws
        del rec
        torch.cuda.empty_cache()
        jm, cm = min(join_ms), min(count_ms)
        rec_bytes = slots * engine.RECORD_BYTES
        line = {
            "workload": f"C5 Tiny-shaped synthetic {N}x{D}, {label}", "epsilon": eps,
            "extra_flags": extra,
            "eps_sq": es, "shard": f"rows {rows[0]}..{rows[1]} ({nrows} points) = rank "
                                   f"{rank} of {world}, x all {N} columns",
            "pairs": pairs, "selectivity": (pairs - nrows) / nrows,
            "join_ms": join_ms, "join_tflops": flops / jm / 1e9,
            "pct_of_sustained": flops / jm / 1e9 / peak_sus if peak_sus else None,
            "pairs_per_s": pairs / (jm / 1e3),
            "count_only_ms": count_ms, "count_only_tflops": flops / cm / 1e9,
            "record_write_cost_ms": jm - cm,
            "records_bytes": rec_bytes,
            "output_write_roofline_ms": rec_bytes / (hbm * 1e9) * 1e3,
            "sort_ms": sort_ms,
            "sort_GBps_records": rec_bytes / (sort_ms / 1e3) / 1e9 if sort_ms else None,
            "eight_gpu_job_tflops_if_balanced": world * flops / jm / 1e9,
            "kernel": L.fasted_join_kernel_name(dd.d_pad, rows[1] - rows[0], dd.n_dev,
                                                jflags).decode(),
            "clocks_join": clk_j.summary(), "clocks_count": clk_c.summary(),
        }
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
