#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "sort or pipeline or long_rows" > gpurun_out/pytest_sort2.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_sort2.log
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/sort_launches_s4096b.csv python scripts/c5_sweep.py --shard 0/8 --reps 1 --only S4096 > gpurun_out/sortprof.log 2>&1
