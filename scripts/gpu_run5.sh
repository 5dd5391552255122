#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python scripts/power_exp.py C4 3 > gpurun_out/power_exp_c4.log 2>&1
timeout 300 python scripts/power_exp.py C3 4 > gpurun_out/power_exp_c3.log 2>&1
timeout 300 python scripts/power_exp.py C2 50 > gpurun_out/power_exp_c2.log 2>&1
