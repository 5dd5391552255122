#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1200 python scripts/tune.py C4 2 "CG=0" "CG=2,G=8192" "CG=2,G=2048" "CG=1,G=2048" "CG=0,G=4096" "CG=0" > gpurun_out/tune_c4_cg2.log 2>&1
