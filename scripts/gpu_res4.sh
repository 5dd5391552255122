#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python scripts/tune.py C3 5 "R=1,CG=2" "R=1,CG=2,F=2" "R=1,CG=2,F=2050" > gpurun_out/tune_c3_count.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:join_tc_res -s 1 -c 1 -o gpurun_out/ncu_c3_res python scripts/ncu_join.py C3 75776 > gpurun_out/ncu_c3.log 2>&1
