#!/bin/bash
# Resident kernel column-segment length (tiles of 256 columns per unit), segment-major + pacing.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python scripts/ab_env.py C3 3 "FASTED_SEG_TILES=64" "FASTED_SEG_TILES=32" "FASTED_SEG_TILES=128" "FASTED_SEG_TILES=256" >> gpurun_out/seg2_ab.txt 2>&1
AB_EPS=7.2300123612099165 AB_SHARD=0/8 timeout 1200 python scripts/ab_env.py C5 2 "FASTED_SEG_TILES=64" "FASTED_SEG_TILES=32" "FASTED_SEG_TILES=128" "FASTED_SEG_TILES=256" >> gpurun_out/seg2_ab.txt 2>&1
AB_EPS=6.896041752764515 AB_SHARD=0/8 timeout 1200 python scripts/ab_env.py C5 2 "FASTED_SEG_TILES=64" "FASTED_SEG_TILES=128" "FASTED_SEG_TILES=256" >> gpurun_out/seg2_ab.txt 2>&1
