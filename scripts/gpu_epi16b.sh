#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "resident" > gpurun_out/pytest_e16.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_e16.log
timeout 900 python scripts/tune.py C3 5 "CG=0,EPI=8" "CG=0,EPI=16" "CG=0,EPI=16,F=2048" "CG=0,EPI=16,F=1024" "CG=0,EPI=8" > gpurun_out/tune_c3_e16.log 2>&1
