#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "multicast or resident or sampled or smoke or sharding" > gpurun_out/pytest_mc.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_mc.log
timeout 1200 python scripts/tune.py C4 2 "CG=1,G=2048" "MC=1,G=2048" "MC=1,G=4096" "MC=1,G=1024" "MC=1,G=2048,F=768" "MC=1,G=2048,F=256" "CG=1,G=2048" "MC=1,G=2048" > gpurun_out/tune_c4_mc.log 2>&1
timeout 600 python scripts/tune.py C2 20 "CG=2,R=0" "MC=1" "CG=1" > gpurun_out/tune_c2_mc.log 2>&1
