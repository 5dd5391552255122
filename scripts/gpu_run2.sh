#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 300 python scripts/debug_c1.py > gpurun_out/debug_c1.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python scripts/prof_join.py C2 2 > gpurun_out/launches_c2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:join_tc -s 2 -c 1 -o gpurun_out/prof_c2 python scripts/prof_join.py C2 3 > gpurun_out/prof_c2.log 2>&1
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 100 > gpurun_out/clocks_c4.csv &
SMI=$!
timeout 300 python scripts/prof_join.py C4 4 > gpurun_out/prof_c4.log 2>&1
kill $SMI
timeout 300 python scripts/prof_join.py C3 3 > gpurun_out/prof_c3.log 2>&1
timeout 300 python scripts/prof_join.py C2 3 exact > gpurun_out/prof_c2_exact.log 2>&1
