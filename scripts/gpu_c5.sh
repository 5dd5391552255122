#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1500 python scripts/c5_sweep.py --shard 0/8 --reps 2 > gpurun_out/c5_sweep.jsonl 2> gpurun_out/c5_sweep.err
