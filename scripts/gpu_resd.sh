#!/bin/bash
# Resident A up to d_pad 512 (default now): GPU suite, memcheck of the new range, C2 + C5 sweep.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
out=gpurun_out/resd.txt
: > $out
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_resd.log 2>&1; tail -2 gpurun_out/pytest_resd.log >> $out
cat > /tmp/san_resd.py <<'PY'
import sys, os
sys.path.insert(0, os.getcwd())
import paper_2508_21230_b200 as F
for n, d, eps in ((2000, 512, 8.6), (1500, 384, 7.7), (999, 300, 6.8)):
    hd = F.to_half(F.generate_synthetic(n, d, seed=n))
    print(n, d, len(F.self_join(hd, eps)), len(F.self_join(hd, eps, symmetric=True)), flush=True)
PY
timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool memcheck python /tmp/san_resd.py 2>&1 | tail -4 >> $out
python scripts/tune.py C2 20 "CG=0" "CG=0" 2>&1 | tail -2 >> $out
timeout 1500 python scripts/c5_sweep.py --shard 0/8 --reps 2 > gpurun_out/c5_resd.jsonl 2>/dev/null
python3 -c "
import json
for l in open('gpurun_out/c5_resd.jsonl'):
    try: d=json.loads(l)
    except Exception: continue
    print(d['workload'][-22:], round(d['join_tflops'],1), 'pairs/s %.3g'%d['pairs_per_s'], 'sort', round(d['sort_ms'],1), d['kernel'], d['clocks_join'].get('sm_mhz'))
" >> $out
cat $out
