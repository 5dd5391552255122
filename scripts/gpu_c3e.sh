#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "resident" > gpurun_out/pytest_c3e.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_c3e.log
timeout 1200 python scripts/tune.py C3 5 "CG=0" "CG=0,F=256" "CG=0,F=2048" "CG=0,F=2" "CG=0" "CG=0,EPI=8" > gpurun_out/tune_c3_e.log 2>&1
