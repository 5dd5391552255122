#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python scripts/power_exp.py C4 3 normal,no-epilogue,load-only,sign-only > gpurun_out/power_exp_c4.log 2>&1
timeout 300 python scripts/power_exp.py C3 4 normal,no-epilogue,load-only,sign-only > gpurun_out/power_exp_c3.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:join_tc -s 9 -c 1 -o gpurun_out/prof_c3 python scripts/prof_join.py C3 2 > gpurun_out/prof_c3.log 2>&1
