#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_lo.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_lo.log
timeout 1200 python bench.py --no-cpu-baseline > gpurun_out/bench_lo.log 2>&1; echo "rc=$?" >> gpurun_out/bench_lo.log
timeout 1500 python scripts/c5_sweep.py --shard 0/8 --reps 1 > gpurun_out/c5_lo.jsonl 2> gpurun_out/c5_lo.err
