#!/bin/bash
# C3 resident-kernel A/B: explicit LOP3 tree (default) vs compiler chain
# (524288), spin waits (8192); hybrid hit search vs per-lane masks on C2/C5.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
out=gpurun_out/ab_tree.txt
: > $out
for k in 1 2; do
  python scripts/tune.py C3 2 "CG=0" "CG=0,F=524288" "CG=0,F=8192" >> $out 2>&1
done
python scripts/tune.py C2 30 "CG=0" "CG=0,F=131072" "CG=0" "CG=0,F=131072" >> $out 2>&1
python scripts/trace_res.py C3 75776 0 > gpurun_out/trace_c3e.txt 2>&1
timeout 900 python -m pytest tests -x -q -m "gpu and not slow" > gpurun_out/pytest_tree.txt 2>&1; tail -2 gpurun_out/pytest_tree.txt >> $out
timeout 900 python scripts/c5_sweep.py --only S4096 --reps 1 --extra-flags 0,131072,0,131072 2>&1 | grep -v "^#" | python3 -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l.strip()); continue
    print(d['workload'][-6:], 'flags', d['extra_flags'], 'join_ms', d['join_ms'], 'count_only_ms', d['count_only_ms'])
" >> $out
cat $out; grep -v "^  t" gpurun_out/trace_c3e.txt
