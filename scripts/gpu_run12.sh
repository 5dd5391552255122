#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
FASTED_CTA_GROUP=2 timeout 600 ncu --set full --clock-control none --import-source on -k regex:join_tc -s 9 -c 1 -o gpurun_out/prof_c2_cg2 python scripts/prof_join.py C2 3 > gpurun_out/prof_c2_cg2.log 2>&1
FASTED_CTA_GROUP=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:join_tc -s 9 -c 1 -o gpurun_out/prof_c2_cg1 python scripts/prof_join.py C2 3 > gpurun_out/prof_c2_cg1.log 2>&1
