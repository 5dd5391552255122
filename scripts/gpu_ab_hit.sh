#!/bin/bash
# Resident kernel A/B: hit warps (default) vs epilogue warps running the rare
# path (FASTED_RES_HIT=0); C3 and C1.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
out=gpurun_out/ab_hit.txt
: > $out
python scripts/tune.py C3 1 "CG=0" > /dev/null 2>&1
for k in 1 2 3; do
  FASTED_RES_HIT=0 python scripts/tune.py C3 2 "CG=0" 2>&1 | sed 's/^/HIT0 /' >> $out
  python scripts/tune.py C3 2 "CG=0" 2>&1 | sed 's/^/HIT2 /' >> $out
done
python scripts/tune.py C3 2 "CG=0,F=2048" "CG=0,F=1024" "CG=0,F=256" 2>&1 | sed 's/^/HIT2 /' >> $out
cat $out
