#!/bin/bash
# A/B: test_wait spin -- 0 none, 3 MMA + producer, 7 MMA + producer + hit warps.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python scripts/ab_env.py C4 4 "FASTED_MMA_SPIN=0" "FASTED_MMA_SPIN=3" "FASTED_MMA_SPIN=7" >> gpurun_out/spin5_ab.txt 2>&1
timeout 600 python scripts/ab_env.py C3 4 "FASTED_MMA_SPIN=0" "FASTED_MMA_SPIN=3" "FASTED_MMA_SPIN=7" >> gpurun_out/spin5_ab.txt 2>&1
AB_EPS=7.049487707996186 AB_SHARD=0/8 timeout 900 python scripts/ab_env.py C5 2 "FASTED_MMA_SPIN=0" "FASTED_MMA_SPIN=3" "FASTED_MMA_SPIN=7" >> gpurun_out/spin5_ab.txt 2>&1
AB_EPS=6.896041752764515 AB_SHARD=0/8 timeout 900 python scripts/ab_env.py C5 2 "FASTED_MMA_SPIN=0" "FASTED_MMA_SPIN=3" "FASTED_MMA_SPIN=7" >> gpurun_out/spin5_ab.txt 2>&1
AB_SHARD=0/8 timeout 900 python scripts/ab_env.py C4 6 "FASTED_MMA_SPIN=0" "FASTED_MMA_SPIN=3" >> gpurun_out/spin5_ab.txt 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit,temperature.gpu --format=csv >> gpurun_out/spin5_ab.txt
