#!/bin/bash
# Round-1 library vs the current product at C5 shard S16 / S4096, C2, C4 (alternating processes).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for lib in paper_2508_21230_b200/libfasted_r1.so paper_2508_21230_b200/libfasted.so paper_2508_21230_b200/libfasted_r1.so paper_2508_21230_b200/libfasted.so; do
  echo "== $lib" >> gpurun_out/r1cmp3.txt
  FASTED_LIB=$lib AB_EPS=6.896041752764515 AB_SHARD=0/8 timeout 900 python scripts/ab_env.py C5 2 "X=0" >> gpurun_out/r1cmp3.txt 2>&1
  FASTED_LIB=$lib AB_EPS=7.2300123612099165 AB_SHARD=0/8 timeout 900 python scripts/ab_env.py C5 2 "X=0" >> gpurun_out/r1cmp3.txt 2>&1
  FASTED_LIB=$lib timeout 900 python scripts/ab_env.py C2 20 "X=0" >> gpurun_out/r1cmp3.txt 2>&1
  FASTED_LIB=$lib timeout 900 python scripts/ab_env.py C4 2 "X=0" >> gpurun_out/r1cmp3.txt 2>&1
done
