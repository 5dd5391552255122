#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "not full_size" > gpurun_out/pytest_lanes.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_lanes.log
timeout 1200 python scripts/tune.py C3 5 "CG=0" "CG=0" "CG=0,F=2" > gpurun_out/tune_c3_lanes.log 2>&1
timeout 1500 python scripts/c5_sweep.py --shard 0/8 --reps 1 --only S > gpurun_out/c5_lanes.jsonl 2> gpurun_out/c5_lanes.err
