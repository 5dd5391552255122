#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "pipeline or symmetric or capacity or sharding or calibration" > gpurun_out/pytest_pipe3.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_pipe3.log
timeout 900 python bench.py --no-accuracy --no-cpu-baseline > gpurun_out/bench_c4_pipe3.log 2>&1
