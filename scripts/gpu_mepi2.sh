#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python scripts/tune.py C2 20 "CG=0,MEPI=8" "CG=0,MEPI=16" "CG=0,MEPI=8" "CG=0,MEPI=16" > gpurun_out/tune_c2_mepi.log 2>&1
timeout 1500 python scripts/tune.py C4 2 "CG=0,MEPI=8" "CG=0,MEPI=16" "CG=0,MEPI=8" "CG=0,MEPI=16" > gpurun_out/tune_c4_mepi.log 2>&1
