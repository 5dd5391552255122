#!/bin/bash
# Re-check of resident-kernel epilogue forms with spin waits + pacing: 16 warps + hit
# warps (SPARSE default), 16 warps staged (FASTED_RES_HIT=0), 8 warps x 128 columns.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python scripts/ab_env.py C3 3 "X=0" "FASTED_RES_HIT=0" "FASTED_RES_EPI=8" >> gpurun_out/forms2_ab.txt 2>&1
AB_EPS=7.1352369182727085 AB_SHARD=0/8 timeout 900 python scripts/ab_env.py C5 2 "X=0" "FASTED_RES_HIT=2" "FASTED_RES_EPI=8" >> gpurun_out/forms2_ab.txt 2>&1
AB_EPS=7.2300123612099165 AB_SHARD=0/8 timeout 900 python scripts/ab_env.py C5 2 "X=0" "FASTED_RES_EPI=8" >> gpurun_out/forms2_ab.txt 2>&1
timeout 600 python scripts/ab_env.py C2 20 "X=0" "FASTED_RES_EPI=8" >> gpurun_out/forms2_ab.txt 2>&1
