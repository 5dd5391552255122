#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python scripts/tune.py C2 20 "CG=0" "CG=2,G=16384" "CG=2,G=8192" "CG=2,G=4096" "CG=0" "CG=2,G=8192" > gpurun_out/tune_c2_pair16.log 2>&1
