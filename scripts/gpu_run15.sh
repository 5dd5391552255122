#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1500 python scripts/tune.py C4 3 "CG=2,G=8192,F=2048" "CG=1,G=2048,F=2048" "CG=2,G=8192,F=2" "CG=1,G=2048,F=2" "CG=2,G=8192" "CG=1,G=2048" > gpurun_out/tune_c4b.log 2>&1
