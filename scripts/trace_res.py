"""Per-tile timeline of the resident-A kernel (FASTED_JOIN_DIAG_TRACE).

CTA 0 stamps SM clock64 at: MMA warp {tempty passed (about to issue tile t),
tfull committed}; each epilogue warp {tfull passed, TMEM loads landed, tempty
arrived, tile done}.  Prints the medians over tiles 16..TRACE_TILES-1 of the
MMA period, the gaps and the epilogue phases, in SM cycles.
usage: python scripts/trace_res.py C3 [rows] [extra_flags,...]
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2508_21230_b200 as F  # noqa: E402
from bench import SEED, WORKLOADS  # noqa: E402
from paper_2508_21230_b200 import _lib, engine  # noqa: E402
# env knobs and diagnostic flags exist only in the experiment build
_lib.LIB_PATH = os.path.abspath(os.environ.get("FASTED_LIB", _lib.EXP_LIB_PATH))

TRACE = 65536
TT, NW = 256, 16
HW, HE = 2, 512                       # hit warps traced, entries each
WORDS = TT * (2 + 8 * NW) + HW * HE * 4

wl = sys.argv[1] if len(sys.argv) > 1 else "C3"
rows = int(sys.argv[2]) if len(sys.argv) > 2 else 148 * 256 * 2
extra = [int(x) for x in sys.argv[3].split(",")] if len(sys.argv) > 3 else [0]
name, n, d, eps = WORKLOADS[wl]
hd = F.to_half(F.generate_synthetic(n, d, seed=SEED))
dd = engine.upload(hd, 0)
es = float(np.float32(np.float32(eps) ** 2))
r = (0, min(rows, dd.n_dev))
L = _lib.load()
print("kernel:", L.fasted_join_kernel_name(dd.d_pad, r[1] - r[0], dd.n_dev, 0).decode())
first = engine.join_device(dd, es, rows=r, sort=False, capacity=(r[1] - r[0]) * 8192)
cap = first.count + engine.hole_slack(0) + WORDS // 2
rec = torch.empty((cap, 4), dtype=torch.int32, device="cuda")
cnt = torch.zeros(2, dtype=torch.int64, device="cuda")
s = torch.cuda.current_stream()
for fl in extra:
    for rep in range(2):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        engine.join_raw(dd, es, fl | TRACE, r, (0, dd.n_dev), rec, cap, cnt, s.cuda_stream)
        e1.record(s)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    tr = rec.view(torch.int64).flatten()[-WORDS:].cpu().numpy().astype(np.int64)
    mma = tr[:2 * TT].reshape(TT, 2)
    epi = tr[2 * TT:TT * (2 + 8 * NW)].reshape(TT, NW, 8)
    hit = tr[TT * (2 + 8 * NW):].reshape(HW, HE, 4)
    lo = 16
    t0 = mma[lo:, 0]
    period = np.diff(t0)
    issue = mma[lo:, 1] - mma[lo:, 0]
    # how long the MMA warp waited for tempty(t): from its previous tile's
    # tfull commit to passing tempty(t)
    mwait = mma[lo:, 0] - mma[lo - 1:-1, 1]
    tf = epi[lo:, :, 0]
    ld = epi[lo:, :, 1] - epi[lo:, :, 0]
    arr = epi[lo:, :, 2] - epi[lo:, :, 1]
    math = epi[lo:, :, 3] - epi[lo:, :, 2]
    # slowest warp's arrive relative to the MMA warp passing tempty two tiles later
    last_arrive = epi[lo:, :, 2].max(axis=1)
    wake = mma[lo + 2:, 0] - last_arrive[:-2]
    # epilogue warp idle: tile done -> next tfull passed
    idle = epi[lo + 1:, :, 0] - epi[lo:-1, :, 3]
    tf_after_commit = tf.min(axis=1) - mma[lo:, 1]

    def q(x):
        return f"p10 {np.percentile(x, 10):7.0f}  p50 {np.percentile(x, 50):7.0f}  " \
               f"p90 {np.percentile(x, 90):7.0f}"

    print(f"\n== {wl} rows {r} flags {fl}: {ms:.3f} ms, "
          f"{2.0 * (r[1] - r[0]) * n * d / ms / 1e9:.1f} TFLOPS, count {int(cnt[0])}")
    print(f"MMA period per tile            {q(period)}")
    print(f"MMA issue (tempty -> commit)   {q(issue)}")
    print(f"MMA wait for tempty            {q(mwait)}")
    print(f"commit -> first tfull seen     {q(tf_after_commit)}")
    print(f"epi: tfull -> loads landed     {q(ld)}")
    print(f"epi: loads -> arrived          {q(arr)}")
    print(f"epi: arrived -> tile done      {q(math)}")
    print(f"epi: tile done -> next tfull   {q(idle)}")
    print(f"last arrive -> MMA past tempty {q(wake)}")
    rare = epi[lo:, :, 7] >= 1
    pushed = epi[lo:, :, 7] > 1     # hit-warp build: [4] after the tail atomic, [7] after the puts
    vote = epi[lo:, :, 4] - epi[lo:, :, 2]
    print(f"epi: arrived -> slice vote     {q(vote)}")
    if rare.any():
        e = epi[lo:][rare]
        print(f"rare slices: {rare.mean() * 100:.1f}% of warp-tiles")
        print(f"  vote -> row loop start       {q(e[:, 5] - e[:, 4])}")
        print(f"  row loop (records appended)  {q(e[:, 6] - e[:, 5])}")
        print(f"  appended -> tile done        {q(e[:, 3] - e[:, 6])}")
        print(f"  arrived -> tile done (rare)  {q(e[:, 3] - e[:, 2])}")
        if pushed.any():
            e2 = epi[lo:][pushed]
            e2 = e2[(e2[:, 4] > e2[:, 5]) & (e2[:, 7] > e2[:, 4]) & (e2[:, 6] >= e2[:, 7])]
            if len(e2):
                print(f"  push: start -> tail atomic   {q(e2[:, 4] - e2[:, 5])}")
                print(f"  push: tail atomic -> puts    {q(e2[:, 7] - e2[:, 4])}")
                print(f"  push: puts -> push end       {q(e2[:, 6] - e2[:, 7])}")
            if os.environ.get("TRACE_SLOT"):   # libfasted_exp_slot.so: [6] = slot known free
                e3 = epi[lo:][pushed]
                e3 = e3[(e3[:, 6] >= e3[:, 4]) & (e3[:, 7] >= e3[:, 6])]
                print(f"  push: tail atomic -> slot ok {q(e3[:, 6] - e3[:, 4])}")
                print(f"  push: slot ok -> puts issued {q(e3[:, 7] - e3[:, 6])}")
        nr = epi[lo:][~rare]
        print(f"  arrived -> tile done (none)  {q(nr[:, 3] - nr[:, 2])}")
    # which epilogue warps see tfull late: per warp (warp index 2 + w, SMSP
    # (2 + w) % 4) the median over tiles of (its tfull stamp - the earliest)
    late = np.median(tf - tf.min(axis=1, keepdims=True), axis=0)
    print("tfull lateness per epi warp (median cycles after the first warp):")
    print("  " + " ".join(f"w{2 + w}:{late[w]:.0f}" for w in range(NW)))
    if hit[:, :, 2].any():
        for h in range(HW):
            e = hit[h]
            e = e[(e[:, 2] > 0) & (e[:, 1] > 0)]
            if len(e) < 32:
                continue
            e = e[16:]
            span = e[-1, 2] - e[0, 0]
            busy = (e[:, 2] - e[:, 1]).sum()
            print(f"hit warp {h}: {len(e)} entries over {span} cycles "
                  f"({span / len(e):.0f} cycles per entry), busy {100.0 * busy / span:.0f}%")
            print(f"  wait for entry               {q(e[:, 1] - e[:, 0])}")
            print(f"  process entry                {q(e[:, 2] - e[:, 1])}")
    print("tiles 40..47 (cycles rel. MMA start of tile 40):")
    base = mma[40, 0]
    for t in range(40, 48):
        e = epi[t]
        print(f"  t{t}: mma {mma[t, 0] - base:7d} {mma[t, 1] - base:7d} | tfull "
              f"{e[:, 0].min() - base:7d}..{e[:, 0].max() - base:7d} ld "
              f"{e[:, 1].min() - base:7d}..{e[:, 1].max() - base:7d} arr "
              f"{e[:, 2].min() - base:7d}..{e[:, 2].max() - base:7d} done "
              f"{e[:, 3].min() - base:7d}..{e[:, 3].max() - base:7d}")
