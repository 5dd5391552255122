#!/bin/bash
# Segment-major unit order: pacing window.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python scripts/ab_env.py C3 4 "FASTED_RES_ORDER=1,FASTED_PACE_W=2" "FASTED_RES_ORDER=1,FASTED_PACE_W=4" "FASTED_RES_ORDER=1,FASTED_PACE_W=8" "FASTED_RES_ORDER=1,FASTED_PACE_W=1" >> gpurun_out/order2_ab.txt 2>&1
AB_EPS=7.2300123612099165 AB_SHARD=0/8 timeout 900 python scripts/ab_env.py C5 2 "FASTED_RES_ORDER=1,FASTED_PACE_W=2" "FASTED_RES_ORDER=1,FASTED_PACE_W=4" "FASTED_RES_ORDER=1,FASTED_PACE_W=8" >> gpurun_out/order2_ab.txt 2>&1
