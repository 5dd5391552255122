#!/bin/bash
# C3 A/B/C: previous commit's build, the C-chain build, the working tree.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
out=gpurun_out/ab3.txt
: > $out
python scripts/tune.py C3 1 "CG=0" > /dev/null 2>&1   # warm the box
for k in 1 2; do
  FASTED_LIB=paper_2508_21230_b200/libfasted_prev.so python scripts/tune.py C3 2 "CG=0" 2>&1 | sed 's/^/PREV  /' >> $out
  FASTED_LIB=paper_2508_21230_b200/libfasted_alt.so python scripts/tune.py C3 2 "CG=0" 2>&1 | sed 's/^/CHAIN /' >> $out
  python scripts/tune.py C3 2 "CG=0" 2>&1 | sed 's/^/TREE  /' >> $out
  FASTED_LIB=paper_2508_21230_b200/libfasted_head.so python scripts/tune.py C3 2 "CG=0" 2>&1 | sed 's/^/HEAD  /' >> $out
done
cat $out
