#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 300 python scripts/debug_sort.py > gpurun_out/debug_sort.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:join_tc -s 9 -c 1 -o gpurun_out/prof_c2b python scripts/prof_join.py C2 3 > gpurun_out/prof_c2b.log 2>&1
timeout 300 python scripts/power_probe.py > gpurun_out/power_probe.log 2>&1
