#!/bin/bash
# A/B vs the HEAD-era build (libfasted_head.so): C5 S4096 shard, C2, C3.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
out=gpurun_out/ab_c5.txt
: > $out
fmt='import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    print(d["workload"][-6:], "join_ms", [round(x,1) for x in d["join_ms"]], "count_only_ms", [round(x,1) for x in d["count_only_ms"]])'
timeout 600 python -m pytest tests/test_gpu.py -x -q -k "append or segmented or resident or multicast or symmetric or low_output" >> $out 2>&1
for k in 1 2; do
  FASTED_LIB=paper_2508_21230_b200/libfasted_head.so timeout 900 python scripts/c5_sweep.py --only S4096 --reps 2 2>/dev/null | python3 -c "$fmt" | sed 's/^/HEAD /' >> $out
  timeout 900 python scripts/c5_sweep.py --only S4096 --reps 2 2>/dev/null | python3 -c "$fmt" | sed 's/^/NEW  /' >> $out
done
for k in 1 2; do
FASTED_LIB=paper_2508_21230_b200/libfasted_head.so timeout 900 python scripts/tune.py C2 30 "CG=0" "CG=0" 2>&1 | sed 's/^/HEAD /' >> $out
timeout 900 python scripts/tune.py C2 30 "CG=0" "CG=0" 2>&1 | sed 's/^/NEW  /' >> $out
done
FASTED_LIB=paper_2508_21230_b200/libfasted_head.so timeout 900 python scripts/tune.py C3 2 "CG=0" "CG=0" 2>&1 | sed 's/^/HEAD /' >> $out
timeout 900 python scripts/tune.py C3 2 "CG=0" "CG=0" 2>&1 | sed 's/^/NEW  /' >> $out
cat $out
