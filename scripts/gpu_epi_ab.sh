#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1200 python scripts/tune.py C3 5 "CG=0,EPI=8" "CG=0,EPI=16" "CG=0,EPI=8" "CG=0,EPI=16" "CG=0,EPI=8" "CG=0,EPI=16" > gpurun_out/tune_c3_epi_ab.log 2>&1
