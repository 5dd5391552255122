#!/bin/bash
# A/B at full C4 size (1.35 s launches, power-capped): MMA warp test_wait spin.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python scripts/ab_env.py C4 8 "FASTED_MMA_SPIN=0" "FASTED_MMA_SPIN=1" >> gpurun_out/mmaspin3_ab.txt 2>&1
AB_EPS=6.896041752764515 AB_SHARD=0/8 timeout 900 python scripts/ab_env.py C5 3 "FASTED_MMA_SPIN=0" "FASTED_MMA_SPIN=1" >> gpurun_out/mmaspin3_ab.txt 2>&1
