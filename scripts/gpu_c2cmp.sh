#!/bin/bash
# C2 (60K x 512): round-1 library vs current product, 100 launches each, alternating processes x3;
# and in-process: pacing / unit order / spin variants on the experiment build.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for r in 1 2 3; do
for lib in paper_2508_21230_b200/libfasted_r1.so paper_2508_21230_b200/libfasted.so; do
  echo "== $lib" >> gpurun_out/c2cmp.txt
  FASTED_LIB=$lib timeout 600 python scripts/ab_env.py C2 100 "X=0" 2>&1 | cut -c1-90 >> gpurun_out/c2cmp.txt
done
done
timeout 600 python scripts/ab_env.py C2 100 "X=0" "FASTED_PACE_W=0" "FASTED_RES_ORDER=0" "FASTED_MMA_SPIN=0" 2>&1 | cut -c1-90 >> gpurun_out/c2cmp.txt
