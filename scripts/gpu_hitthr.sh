#!/bin/bash
# Hit warps vs staged writers at C5 S~256 / S~1024 under segment-major + pacing (SPARSE threshold check).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
AB_EPS=7.049487707996186 AB_SHARD=0/8 timeout 900 python scripts/ab_env.py C5 2 "FASTED_RES_HIT=2" "FASTED_RES_HIT=0" >> gpurun_out/hitthr_ab.txt 2>&1
AB_EPS=7.1352369182727085 AB_SHARD=0/8 timeout 900 python scripts/ab_env.py C5 2 "FASTED_RES_HIT=2" "FASTED_RES_HIT=0" >> gpurun_out/hitthr_ab.txt 2>&1
timeout 900 python scripts/ab_env.py C3 3 "FASTED_RES_HIT=2" "FASTED_RES_HIT=0" >> gpurun_out/hitthr_ab.txt 2>&1
