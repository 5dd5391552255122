#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "low_output or resident or symmetric" > gpurun_out/pytest_sepi.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_sepi.log
timeout 1500 python scripts/tune.py C4 2 "CG=2,G=16384,SEPI=8" "CG=2,G=16384,SEPI=16" "CG=2,G=16384,SEPI=8" "CG=2,G=16384,SEPI=16" > gpurun_out/tune_c4_sepi.log 2>&1
