#!/bin/bash
# Round-1 library vs the current product (segment-major + pacing), C3 full and shard, alternating processes.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for r in 1 2; do
for lib in paper_2508_21230_b200/libfasted_r1.so paper_2508_21230_b200/libfasted.so; do
  echo "== $lib" >> gpurun_out/r1cmp2.txt
  FASTED_LIB=$lib timeout 900 python scripts/ab_env.py C3 3 "X=0" >> gpurun_out/r1cmp2.txt 2>&1
  FASTED_LIB=$lib AB_SHARD=0/8 timeout 900 python scripts/ab_env.py C3 5 "X=0" >> gpurun_out/r1cmp2.txt 2>&1
done
done
