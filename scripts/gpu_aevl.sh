#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1500 python scripts/tune.py C4 2 "CG=2,G=16384" "CG=2,G=16384,F=32768" "CG=2,G=16384" "CG=2,G=16384,F=32768" "CG=2,G=24576" "CG=2,G=12288" > gpurun_out/tune_c4_aevl.log 2>&1
