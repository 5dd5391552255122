#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python scripts/tune.py C3 5 "CG=0" "CG=0,F=16384" "CG=0,F=17408" "CG=0,F=1024" "CG=0,F=256" > gpurun_out/tune_c3_ldx64.log 2>&1
