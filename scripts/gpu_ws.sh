#!/bin/bash
# Staged-writer buffer size in the resident kernel (records per warp buffer 16 -> 32),
# dense output: C5 shard S~4096 / S~1024, C2; alternating processes.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
P=paper_2508_21230_b200
for r in 1 2; do
for lib in libfasted_exp libfasted_exp_ws512; do
  echo "== $lib" >> gpurun_out/ws_ab.txt
  FASTED_LIB=$P/$lib.so AB_EPS=7.2300123612099165 AB_SHARD=0/8 timeout 900 python scripts/ab_env.py C5 2 "X=0" >> gpurun_out/ws_ab.txt 2>&1
  FASTED_LIB=$P/$lib.so AB_EPS=7.1352369182727085 AB_SHARD=0/8 timeout 900 python scripts/ab_env.py C5 2 "X=0" >> gpurun_out/ws_ab.txt 2>&1
  FASTED_LIB=$P/$lib.so timeout 900 python scripts/ab_env.py C2 50 "X=0" >> gpurun_out/ws_ab.txt 2>&1
done
done
