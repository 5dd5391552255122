#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "not c3_full" > gpurun_out/pytest_elect.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_elect.log
timeout 1200 python scripts/tune.py C4 2 "MC=1,G=4096" "MC=1,G=8192" "CG=1,G=2048" "MC=1,G=8192,F=256" > gpurun_out/tune_c4_elect.log 2>&1
timeout 900 python scripts/tune.py C3 5 "CG=2" "CG=2,F=256" "CG=2,F=2050" > gpurun_out/tune_c3_elect.log 2>&1
timeout 600 python scripts/tune.py C2 20 "CG=2,R=0" "MC=1" "CG=1" > gpurun_out/tune_c2_elect.log 2>&1
