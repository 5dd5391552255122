#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_c4.log 2>&1; echo "rc=$?" >> gpurun_out/bench_c4.log
timeout 900 python -m pytest tests -m "gpu and slow" -x -q -s > gpurun_out/pytest_slow.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_slow.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 > gpurun_out/launches_c4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:join_tc -s 9 -c 1 -o gpurun_out/prof_c4 python scripts/prof_join.py C4 2 > gpurun_out/prof_c4.log 2>&1
