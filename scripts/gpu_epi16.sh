#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "resident or tc or smoke" > gpurun_out/pytest_epi.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_epi.log
timeout 900 python scripts/tune.py C3 5 "CG=2,EPI=8" "CG=2,EPI=16" "CG=2,EPI=16,F=2050" "CG=2,EPI=16,F=256" "CG=2,EPI=16,F=2" > gpurun_out/tune_c3_epi16.log 2>&1
