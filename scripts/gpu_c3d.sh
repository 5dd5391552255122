#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1200 python scripts/tune.py C3 5 "CG=0" "CG=0,F=256" "CG=0,F=1024" "CG=0,F=2048" "CG=0,F=2" "CG=0" > gpurun_out/tune_c3_d.log 2>&1
