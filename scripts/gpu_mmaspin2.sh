#!/bin/bash
# A/B: MMA warp test_wait spin at C4 (CTA-pair streaming kernel) and C3/C2 (resident).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for r in 1 2; do
AB_SHARD=0/8 timeout 600 python scripts/ab_env.py C4 5 "FASTED_MMA_SPIN=0" "FASTED_MMA_SPIN=1" >> gpurun_out/mmaspin2_ab.txt 2>&1
timeout 600 python scripts/ab_env.py C3 4 "FASTED_MMA_SPIN=0" "FASTED_MMA_SPIN=1" >> gpurun_out/mmaspin2_ab.txt 2>&1
done
timeout 600 python scripts/ab_env.py C2 30 "FASTED_MMA_SPIN=0" "FASTED_MMA_SPIN=1" >> gpurun_out/mmaspin2_ab.txt 2>&1
