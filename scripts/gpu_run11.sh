#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
FASTED_CTA_GROUP=1 timeout 900 python -m pytest tests -m "gpu and not slow" -x -q -k "tc or sampled or smoke or loaded" > gpurun_out/pytest_gpu_cg1.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_cg1.log
timeout 900 python scripts/tune.py C4 3 "CG=2,G=8192" "CG=1,G=2048" "CG=2,G=32768" "CG=2,G=4096" "CG=2,G=8192,F=256" > gpurun_out/tune_c4.log 2>&1
timeout 600 python scripts/tune.py C3 4 "CG=2,G=8192" "CG=1,G=2048" "CG=2,G=32768" "CG=2,G=8192,F=256" > gpurun_out/tune_c3.log 2>&1
timeout 300 python scripts/tune.py C2 50 "CG=2,G=8192" "CG=1,G=2048" "CG=2,G=2048" "CG=2,G=8192,F=256" > gpurun_out/tune_c2.log 2>&1
