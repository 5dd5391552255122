#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "not full_size" > gpurun_out/pytest_c3c.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_c3c.log
timeout 900 python scripts/tune.py C3 5 "CG=0" "CG=0,F=2048" "CG=0,F=2" "CG=0,F=1024" > gpurun_out/tune_c3_c.log 2>&1
timeout 900 python scripts/tune.py C4 2 "CG=0" > gpurun_out/tune_c4_c.log 2>&1
timeout 900 python scripts/tune.py C2 20 "CG=0" > gpurun_out/tune_c2_c.log 2>&1
