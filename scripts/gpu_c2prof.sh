#!/bin/bash
# C2 (60K x 512) per-launch breakdown: join vs Gram pre-pass vs augment prep, and the
# join kernel's tensor-pipe activity / L2 traffic.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed,lts__t_sectors_srcunit_tex.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,lts__t_sector_hit_rate.pct,dram__bytes_read.sum,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:join_tc_res -s 6 -c 3 --csv --log-file gpurun_out/c2prof.csv python scripts/ab_env.py C2 3 "X=0" > gpurun_out/c2prof.log 2>&1
timeout 600 nsys --version > /dev/null 2>&1 || true
timeout 600 python - > gpurun_out/c2_wall.txt 2>&1 <<'PY'
import os, sys, time, statistics
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2508_21230_b200 as F
from bench import SEED, WORKLOADS
from paper_2508_21230_b200 import _lib, engine
name, n, d, eps = WORKLOADS["C2"]
hd = F.to_half(F.generate_synthetic(n, d, seed=SEED)); dd = engine.upload(hd, 0)
es = float(np.float32(np.float32(eps) ** 2))
rows = (0, dd.n_dev)
first = engine.join_device(dd, es, rows=rows, sort=False); cap = first.count + engine.hole_slack(0)
rec = torch.empty((cap, 4), dtype=torch.int32, device="cuda"); cnt = torch.zeros(2, dtype=torch.int64, device="cuda")
s = torch.cuda.current_stream()
fl = _lib.JOIN_TC | engine.form_hints(first.count, rows, (0, dd.n_dev))
for it in range(3):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(51)]
    ev[0].record(s)
    for k in range(50):
        engine.join_raw(dd, es, fl, rows, (0, dd.n_dev), rec, cap, cnt, s.cuda_stream); ev[k+1].record(s)
    torch.cuda.synchronize()
    t = [ev[k].elapsed_time(ev[k+1]) for k in range(50)]
    print("back-to-back 50: median %.3f ms min %.3f max %.3f" % (statistics.median(t), min(t), max(t)))
PY
