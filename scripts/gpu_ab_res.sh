#!/bin/bash
# A/B of an epilogue change: HEAD build (libfasted_head.so) vs the working
# tree, alternating processes; then the GPU suite and a resident-kernel trace.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
out=gpurun_out/ab_res.txt
: > $out
for k in 1 2; do
  FASTED_LIB=paper_2508_21230_b200/libfasted_head.so python scripts/tune.py C3 3 "CG=0" 2>&1 | sed 's/^/HEAD /' >> $out
  python scripts/tune.py C3 3 "CG=0" 2>&1 | sed 's/^/NEW  /' >> $out
done
FASTED_LIB=paper_2508_21230_b200/libfasted_head.so python scripts/tune.py C2 20 "CG=0" 2>&1 | sed 's/^/HEAD /' >> $out
python scripts/tune.py C2 20 "CG=0" 2>&1 | sed 's/^/NEW  /' >> $out
FASTED_LIB=paper_2508_21230_b200/libfasted_head.so python scripts/tune.py C4 1 "CG=0,F=8" 2>&1 | sed 's/^/HEAD /' >> $out
python scripts/tune.py C4 1 "CG=0,F=8" 2>&1 | sed 's/^/NEW  /' >> $out
python scripts/trace_res.py C3 75776 0 > gpurun_out/trace_c3d.txt 2>&1
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_ab.txt 2>&1; tail -3 gpurun_out/pytest_ab.txt >> $out
FASTED_LIB=paper_2508_21230_b200/libfasted_head.so timeout 600 python scripts/c5_sweep.py --only S4096 --reps 1 2>&1 | grep -v "^#" | sed 's/^/HEAD /' >> $out
timeout 600 python scripts/c5_sweep.py --only S4096 --reps 1 2>&1 | grep -v "^#" | sed 's/^/NEW  /' >> $out
cat $out | cut -c1-400; grep -v "^  t" gpurun_out/trace_c3d.txt
