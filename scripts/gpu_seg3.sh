#!/bin/bash
# Segment length for single-buffered A panels (d >= 384): 64 vs 128 vs 256 tiles per unit.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python scripts/ab_env.py C2 60 "FASTED_SEG_TILES=64" "FASTED_SEG_TILES=128" "FASTED_SEG_TILES=256" >> gpurun_out/seg3_ab.txt 2>&1
for e in 6.896041752764515 7.1352369182727085 0.0; do
AB_EPS=$e AB_SHARD=0/8 timeout 1200 python scripts/ab_env.py C5 2 "FASTED_SEG_TILES=64" "FASTED_SEG_TILES=128" "FASTED_SEG_TILES=256" >> gpurun_out/seg3_ab.txt 2>&1
done
