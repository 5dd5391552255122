#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
FASTED_CTA_GROUP=1 FASTED_GROUP_ROWS=2048 timeout 1500 python scripts/c5_sweep.py --shard 0/8 --reps 1 --only S4096 > gpurun_out/c5_cg1.jsonl 2> gpurun_out/c5_cg1.err
FASTED_CTA_GROUP=1 FASTED_GROUP_ROWS=2048 timeout 1500 python scripts/c5_sweep.py --shard 0/8 --reps 1 --only S0 >> gpurun_out/c5_cg1.jsonl 2>> gpurun_out/c5_cg1.err
