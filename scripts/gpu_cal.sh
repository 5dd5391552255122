#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -s -k "calibration" > gpurun_out/pytest_cal.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_cal.log
timeout 600 python -m paper_2508_21230_b200.cli calibrate --synthetic 1000000x960 --target-selectivity 64 --calibration-method device --calibration-tol 0.01 --json > gpurun_out/cal_c4.json 2>&1
