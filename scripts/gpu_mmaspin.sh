#!/bin/bash
# A/B: MMA warp waits (accumulator release, B stages) by try_wait suspend vs test_wait spin.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for r in 1 2 3; do
AB_SHARD=0/8 timeout 600 python scripts/ab_env.py C3 6 "FASTED_MMA_SPIN=0" "FASTED_MMA_SPIN=1" "FASTED_MMA_SPIN=0,F=256" "FASTED_MMA_SPIN=1,F=256" >> gpurun_out/mmaspin_ab.txt 2>&1
done
timeout 600 python scripts/ab_env.py C2 20 "FASTED_MMA_SPIN=0" "FASTED_MMA_SPIN=1" >> gpurun_out/mmaspin_ab.txt 2>&1
FASTED_MMA_SPIN=1 FASTED_RES_HIT=2 timeout 300 python scripts/trace_res.py C3 75776 256 > gpurun_out/mmaspin_trace.txt 2>&1
FASTED_MMA_SPIN=1 FASTED_RES_HIT=2 timeout 300 python scripts/trace_res.py C3 75776 0 >> gpurun_out/mmaspin_trace.txt 2>&1
