#!/bin/bash
# C4 raster group re-check with pacing (FASTED_GROUP_ROWS).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1500 python scripts/ab_env.py C4 3 "FASTED_GROUP_ROWS=16384" "FASTED_GROUP_ROWS=32768" "FASTED_GROUP_ROWS=8192" "FASTED_GROUP_ROWS=65536" >> gpurun_out/raster_ab.txt 2>&1
