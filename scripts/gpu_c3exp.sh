#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python scripts/tune.py C3 5 "CG=2" "CG=2,F=256" "CG=2,F=1024" "CG=2,F=2048" "CG=2,F=8192" "CG=2,F=9216" "CG=2" > gpurun_out/tune_c3_exp.log 2>&1
timeout 900 python scripts/tune.py C4 2 "MC=1" "MC=1,F=8192" > gpurun_out/tune_c4_spin.log 2>&1
