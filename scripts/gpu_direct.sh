#!/bin/bash
# A/B: resident-kernel rare path -- hit warps (product for SPARSE) vs staged
# writers (FASTED_RES_HIT=0) vs the direct register->global writer
# (FASTED_RES_DIRECT=1); C3 shard 0/8 and C2.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for r in 1 2 3; do
AB_SHARD=0/8 timeout 600 python scripts/ab_env.py C3 6 "X=0" "FASTED_RES_DIRECT=1" "FASTED_RES_HIT=0" >> gpurun_out/direct_ab.txt 2>&1
done
timeout 600 python scripts/ab_env.py C2 20 "X=0" "FASTED_RES_DIRECT=1" "FASTED_RES_HIT=0" >> gpurun_out/direct_ab.txt 2>&1
