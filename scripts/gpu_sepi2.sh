#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 2000 python scripts/tune.py C4 2 "CG=2,G=16384,SEPI=8" "CG=2,G=16384,SEPI=16" "CG=2,G=16384,SEPI=8" "CG=2,G=16384,SEPI=16" "CG=2,G=16384,SEPI=8" "CG=2,G=16384,SEPI=16" > gpurun_out/tune_c4_sepi2.log 2>&1
FASTED_STREAM_EPI=16 timeout 1500 python scripts/c5_sweep.py --shard 0/8 --reps 1 --only S > gpurun_out/c5_sepi16.jsonl 2> gpurun_out/c5_sepi16.err
FASTED_STREAM_EPI=8 timeout 1500 python scripts/c5_sweep.py --shard 0/8 --reps 1 --only S > gpurun_out/c5_sepi8.jsonl 2> gpurun_out/c5_sepi8.err
