#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:join_tc -s 9 -c 1 -o gpurun_out/prof_c2c python scripts/prof_join.py C2 3 > gpurun_out/prof_c2c.log 2>&1
