#!/bin/bash
# A/B: hit queue of 16 (libfasted_exp.so) vs 32 slots (libfasted_exp_q32.so), C3 shard 0/8.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for r in 1 2 3; do
for lib in paper_2508_21230_b200/libfasted_exp.so paper_2508_21230_b200/libfasted_exp_q32.so; do
  echo "== $lib" >> gpurun_out/q32_ab.txt
  FASTED_LIB=$lib AB_SHARD=0/8 timeout 600 python scripts/ab_env.py C3 5 "X=0" >> gpurun_out/q32_ab.txt 2>&1
done
done
FASTED_LIB=paper_2508_21230_b200/libfasted_exp_q32.so FASTED_RES_HIT=2 timeout 300 python scripts/trace_res.py C3 75776 0 > gpurun_out/q32_trace.txt 2>&1
