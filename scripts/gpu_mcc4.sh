#!/bin/bash
# C4 with pacing: CTA pair (product) vs B-multicast clusters (paced / unpaced).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1500 python scripts/ab_env.py C4 3 "X=0" "FASTED_PAIR_LOWOUT=0,FASTED_MC_PACE_W=1" "FASTED_PAIR_LOWOUT=0,FASTED_MC_PACE_W=0" >> gpurun_out/mcc4_ab.txt 2>&1
