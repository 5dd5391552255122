#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
FASTED_CTA_GROUP=2 FASTED_GROUP_ROWS=16384 timeout 1500 python scripts/c5_sweep.py --shard 0/8 --reps 1 --only S > gpurun_out/c5_cg2.jsonl 2> gpurun_out/c5_cg2.err
timeout 1200 python scripts/tune.py C3 5 "CG=0" "CG=2,R=0,G=16384" "CG=2,R=0,G=8192" > gpurun_out/tune_c3_cg2.log 2>&1
