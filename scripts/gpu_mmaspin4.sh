#!/bin/bash
# A/B: test_wait spin for the MMA warp (1), the producer (2), both (3), vs try_wait suspend (0).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python scripts/ab_env.py C4 5 "FASTED_MMA_SPIN=0" "FASTED_MMA_SPIN=1" "FASTED_MMA_SPIN=3" >> gpurun_out/mmaspin4_ab.txt 2>&1
AB_EPS=6.896041752764515 AB_SHARD=0/8 timeout 900 python scripts/ab_env.py C5 3 "FASTED_MMA_SPIN=0" "FASTED_MMA_SPIN=1" "FASTED_MMA_SPIN=3" >> gpurun_out/mmaspin4_ab.txt 2>&1
AB_EPS=7.2300123612099165 AB_SHARD=0/8 timeout 900 python scripts/ab_env.py C5 2 "FASTED_MMA_SPIN=0" "FASTED_MMA_SPIN=1" "FASTED_MMA_SPIN=3" >> gpurun_out/mmaspin4_ab.txt 2>&1
timeout 600 python scripts/ab_env.py C3 4 "FASTED_MMA_SPIN=0" "FASTED_MMA_SPIN=1" "FASTED_MMA_SPIN=3" >> gpurun_out/mmaspin4_ab.txt 2>&1
timeout 600 python scripts/ab_env.py C2 30 "FASTED_MMA_SPIN=0" "FASTED_MMA_SPIN=1" "FASTED_MMA_SPIN=3" >> gpurun_out/mmaspin4_ab.txt 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit,temperature.gpu --format=csv >> gpurun_out/mmaspin4_ab.txt
