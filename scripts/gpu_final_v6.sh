#!/bin/bash
# Final validation of the last commit: GPU suite, smoke, bench + reference arm, and an in-process
# check that pacing is active (paced vs unpaced C3 and C4 shard).
cd "$(dirname "$0")/.."
bash scripts/gpu_r2.sh
timeout 900 python scripts/ab_env.py C3 3 "FASTED_PACE_W=2" "FASTED_PACE_W=0" > gpurun_out/v6_pace_check.txt 2>&1
AB_SHARD=0/8 timeout 900 python scripts/ab_env.py C4 3 "FASTED_STREAM_PACE_W=1" "FASTED_STREAM_PACE_W=0" >> gpurun_out/v6_pace_check.txt 2>&1
