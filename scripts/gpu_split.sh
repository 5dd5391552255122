#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
FASTED_SPLIT_ISSUE=1 timeout 600 python -m pytest tests -m gpu -x -q -k "resident or smoke or c1_tc" > gpurun_out/pytest_split.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_split.log
timeout 900 python scripts/tune.py C3 5 "CG=0" "CG=0,SPLIT=1" "CG=0" "CG=0,SPLIT=1" "CG=0,SPLIT=1,F=2048" > gpurun_out/tune_c3_split.log 2>&1
