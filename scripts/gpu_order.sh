#!/bin/bash
# Resident-kernel unit order: row-tile rounds (product) vs segment-major (round-1 order), paced.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python scripts/ab_env.py C3 4 "FASTED_RES_ORDER=0" "FASTED_RES_ORDER=1" "FASTED_RES_ORDER=1,FASTED_PACE_W=0" >> gpurun_out/order_ab.txt 2>&1
AB_EPS=7.2300123612099165 AB_SHARD=0/8 timeout 900 python scripts/ab_env.py C5 2 "FASTED_RES_ORDER=0" "FASTED_RES_ORDER=1" >> gpurun_out/order_ab.txt 2>&1
AB_EPS=6.896041752764515 AB_SHARD=0/8 timeout 900 python scripts/ab_env.py C5 2 "FASTED_RES_ORDER=0" "FASTED_RES_ORDER=1" >> gpurun_out/order_ab.txt 2>&1
AB_EPS=7.1352369182727085 AB_SHARD=0/8 timeout 900 python scripts/ab_env.py C5 2 "FASTED_RES_ORDER=0" "FASTED_RES_ORDER=1" >> gpurun_out/order_ab.txt 2>&1
timeout 600 python scripts/ab_env.py C2 30 "FASTED_RES_ORDER=0" "FASTED_RES_ORDER=1" >> gpurun_out/order_ab.txt 2>&1
for o in 0 1; do FASTED_RES_ORDER=$o timeout 900 python scripts/c5_sweep.py --shard 0/8 --reps 1 --only S4096 >> gpurun_out/order_c5sort.jsonl 2>&1; done
