#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
export FASTED_GROUP_ROWS=4096
timeout 600 ncu --set full --clock-control none --import-source on -k regex:join_tc_mc -s 1 -c 1 -o gpurun_out/ncu_c4_mc python scripts/ncu_join.py C4 75776 > gpurun_out/ncu_c4.log 2>&1
timeout 900 python scripts/tune.py C4 2 "MC=1,G=4096" "MC=1,G=8192" "MC=1,G=16384" "MC=1,G=4096,F=2" > gpurun_out/tune_c4_mc2.log 2>&1
