#!/bin/bash
# Spin waits re-checked with pacing: C4 full, C3, C5 S16 shard.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1500 python scripts/ab_env.py C4 3 "FASTED_MMA_SPIN=3" "FASTED_MMA_SPIN=0" "FASTED_MMA_SPIN=1" "FASTED_MMA_SPIN=2" >> gpurun_out/spin6_ab.txt 2>&1
timeout 900 python scripts/ab_env.py C3 3 "FASTED_MMA_SPIN=3" "FASTED_MMA_SPIN=0" "FASTED_MMA_SPIN=7" >> gpurun_out/spin6_ab.txt 2>&1
AB_EPS=6.896041752764515 AB_SHARD=0/8 timeout 900 python scripts/ab_env.py C5 2 "FASTED_MMA_SPIN=3" "FASTED_MMA_SPIN=0" "FASTED_MMA_SPIN=7" >> gpurun_out/spin6_ab.txt 2>&1
