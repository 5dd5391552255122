#!/bin/bash
# Resident-kernel pacing window: 1 vs 2 (default) vs 3 layers; C4 streaming window 1 vs 2.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python scripts/ab_env.py C3 4 "FASTED_PACE_W=1" "FASTED_PACE_W=2" "FASTED_PACE_W=3" >> gpurun_out/rpace_ab.txt 2>&1
AB_EPS=7.2300123612099165 AB_SHARD=0/8 timeout 900 python scripts/ab_env.py C5 2 "FASTED_PACE_W=1" "FASTED_PACE_W=2" >> gpurun_out/rpace_ab.txt 2>&1
AB_EPS=6.896041752764515 AB_SHARD=0/8 timeout 900 python scripts/ab_env.py C5 2 "FASTED_PACE_W=1" "FASTED_PACE_W=2" >> gpurun_out/rpace_ab.txt 2>&1
timeout 1200 python scripts/ab_env.py C4 3 "FASTED_STREAM_PACE_W=1" "FASTED_STREAM_PACE_W=2" "FASTED_STREAM_PACE_W=0" >> gpurun_out/rpace_ab.txt 2>&1
