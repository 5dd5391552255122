#!/bin/bash
# Multicast-kernel pacing A/B: C4 rows 0..62.5K (1/16 shard, below 2^36 pairs examined: the mc form).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
AB_SHARD=0/16 timeout 900 python scripts/ab_env.py C4 6 "FASTED_MC_PACE_W=0" "FASTED_MC_PACE_W=1" "FASTED_MC_PACE_W=2" >> gpurun_out/mcpace_ab.txt 2>&1
