#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "resident or tc or sampled or smoke or sharding or capacity or eps_zero or duplicates" > gpurun_out/pytest_res.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_res.log
timeout 900 python scripts/tune.py C3 5 "R=1,CG=2" "R=1,CG=2,F=4096" "R=1,CG=2,F=2048" "R=1,CG=2,F=256" > gpurun_out/tune_c3_lane.log 2>&1
timeout 600 python scripts/tune.py C4 2 "R=1" > gpurun_out/tune_c4_lane.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:join_tc_res -s 1 -c 1 -o gpurun_out/ncu_c3_res python scripts/ncu_join.py C3 75776 > gpurun_out/ncu_c3.log 2>&1
