#!/bin/bash
# Round-1 library (commit 071af31, built from its own sources) vs the current product, same box.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for r in 1 2; do
for lib in paper_2508_21230_b200/libfasted_r1.so paper_2508_21230_b200/libfasted.so; do
  echo "== $lib" >> gpurun_out/r1cmp.txt
  FASTED_LIB=$lib timeout 900 python scripts/ab_env.py C3 3 "X=0" >> gpurun_out/r1cmp.txt 2>&1
  FASTED_LIB=$lib AB_SHARD=0/8 timeout 900 python scripts/ab_env.py C3 5 "X=0" >> gpurun_out/r1cmp.txt 2>&1
done
done
nvidia-smi --query-gpu=clocks.sm,power.draw --format=csv >> gpurun_out/r1cmp.txt
