#!/bin/bash
# Does the 5 ms pacing give-up ever fire in a normal launch? 5 ms vs ~20 s (never), in-process.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python scripts/ab_env.py C3 3 "FASTED_PACE_GIVEUP_US=5000" "FASTED_PACE_GIVEUP_US=2000000000" "FASTED_PACE_W=0" >> gpurun_out/giveup_ab.txt 2>&1
timeout 1200 python scripts/ab_env.py C4 2 "FASTED_PACE_GIVEUP_US=5000" "FASTED_PACE_GIVEUP_US=2000000000" "FASTED_STREAM_PACE_W=0" >> gpurun_out/giveup_ab.txt 2>&1
