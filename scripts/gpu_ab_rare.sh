#!/bin/bash
# A/B of the epilogue hit search: transposed rows (0), per-lane masks
# (131072), hybrid (262144); C2, C3 and a C5 shard at S ~ 4096 and S ~ 250.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
out=gpurun_out/ab_rare.txt
: > $out
for k in 1 2; do
  python scripts/tune.py C2 30 "CG=0" "CG=0,F=131072" "CG=0,F=262144" >> $out 2>&1
  python scripts/tune.py C3 2 "CG=0" "CG=0,F=131072" "CG=0,F=262144" >> $out 2>&1
done
timeout 900 python scripts/c5_sweep.py --only S4096 --reps 1 --extra-flags 0,131072,262144,0,131072,262144 2>&1 | grep -v "^#" | python3 -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l.strip()); continue
    print(d['workload'][-6:], 'flags', d['extra_flags'], 'join_ms', d['join_ms'], 'count_only_ms', d['count_only_ms'])
" >> $out
timeout 600 python scripts/c5_sweep.py --only S256 --reps 1 --extra-flags 0,131072,262144 2>&1 | grep -v "^#" | python3 -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l.strip()); continue
    print(d['workload'][-6:], 'flags', d['extra_flags'], 'join_ms', d['join_ms'], 'kernel', d['kernel'])
" >> $out
cat $out
