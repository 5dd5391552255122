#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1200 python scripts/tune.py C4 2 "CG=1,G=2048" "CG=2,G=2048" "CG=2,G=8192" "CG=1,G=2048,F=768" "CG=2,G=2048,F=768" "CG=1,G=2048,F=256" "CG=2,G=2048,F=256" "CG=1,G=2048" "CG=2,G=2048" > gpurun_out/tune_c4_power.log 2>&1
