#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "not c3_full" > gpurun_out/pytest_sort.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_sort.log
timeout 1500 python scripts/c5_sweep.py --shard 0/8 --reps 1 --only S > gpurun_out/c5_sweep2.jsonl 2> gpurun_out/c5_sweep2.err
