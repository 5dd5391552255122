#!/bin/bash
# StagedWriter without the held L2 policy and with a 32-bit running count (fewer spills in the
# staged-writer epilogues) vs the previous build; alternating processes.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
P=paper_2508_21230_b200
for r in 1 2; do
for lib in libfasted_exp_prev libfasted_exp_lean; do
  echo "== $lib" >> gpurun_out/lean_ab.txt
  FASTED_LIB=$P/$lib.so AB_EPS=7.2300123612099165 AB_SHARD=0/8 timeout 900 python scripts/ab_env.py C5 2 "X=0" >> gpurun_out/lean_ab.txt 2>&1
  FASTED_LIB=$P/$lib.so AB_EPS=7.1352369182727085 AB_SHARD=0/8 timeout 900 python scripts/ab_env.py C5 2 "X=0" >> gpurun_out/lean_ab.txt 2>&1
  FASTED_LIB=$P/$lib.so timeout 900 python scripts/ab_env.py C2 50 "X=0" >> gpurun_out/lean_ab.txt 2>&1
done
done
