#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "multicast" > gpurun_out/pytest_mepi.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_mepi.log
FASTED_MC_EPI=8 timeout 1500 python scripts/c5_sweep.py --shard 0/8 --reps 1 --only S > gpurun_out/c5_mepi8.jsonl 2> gpurun_out/c5_mepi8.err
FASTED_MC_EPI=16 timeout 1500 python scripts/c5_sweep.py --shard 0/8 --reps 1 --only S > gpurun_out/c5_mepi16.jsonl 2> gpurun_out/c5_mepi16.err
