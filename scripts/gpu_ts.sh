#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "tmem_a" > gpurun_out/pytest_ts.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_ts.log
timeout 1200 python scripts/tune.py C3 5 "CG=0" "CG=0,TS=1" "CG=0" "CG=0,TS=1" "CG=0,TS=1,F=256" "CG=0,TS=1,F=2048" > gpurun_out/tune_c3_ts.log 2>&1
