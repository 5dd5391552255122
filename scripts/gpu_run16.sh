#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m "gpu and not slow" -x -q -k "tc or smoke or sampled" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 1500 python scripts/tune.py C4 3 "CG=2,G=8192,F=2" "CG=2,G=8192,F=4098" "CG=2,G=8192,F=4096" "CG=1,G=2048,F=4096" "CG=2,G=8192,F=2048" "CG=1,G=2048" > gpurun_out/tune_c4c.log 2>&1
