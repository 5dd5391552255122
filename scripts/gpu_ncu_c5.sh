#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:join_tc_mc -s 1 -c 1 -o gpurun_out/ncu_c5_s4096 python scripts/ncu_join.py C5 37888 0 7.2300123612099165 > gpurun_out/ncu_c5.log 2>&1
