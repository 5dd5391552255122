#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "resident or multicast or symmetric or smoke" > gpurun_out/pytest_cs.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_cs.log
timeout 900 python scripts/tune.py C3 5 "CG=2" "CG=2,F=2" > gpurun_out/tune_c3_cs.log 2>&1
timeout 1500 python scripts/c5_sweep.py --shard 0/8 --reps 1 --only S4096 > gpurun_out/c5_cs.jsonl 2> gpurun_out/c5_cs.err
