#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python bench.py --no-accuracy --no-cpu-baseline > gpurun_out/bench_c4_pipe2.log 2>&1
