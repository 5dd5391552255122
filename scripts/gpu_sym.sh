#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "symmetric" > gpurun_out/pytest_sym.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_sym.log
timeout 900 python -m pytest tests -m gpu -x -q -k "not c3_full and not symmetric" > gpurun_out/pytest_all.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_all.log
timeout 900 python bench.py --no-accuracy --no-cpu-baseline > gpurun_out/bench_sym.log 2>&1
