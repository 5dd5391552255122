#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1500 python scripts/tune.py C4 2 "CG=0" "CG=2,G=8192" "CG=2,G=16384" "CG=2,G=32768" "CG=0" "CG=2,G=65536" "CG=2,G=16384" "CG=0" > gpurun_out/tune_c4_cg2b.log 2>&1
timeout 600 python scripts/tune.py C2 20 "CG=0" "CG=2,G=8192" "CG=2,G=16384" > gpurun_out/tune_c2_cg2b.log 2>&1
