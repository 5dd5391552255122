#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 300 python scripts/debug_sort.py > gpurun_out/debug_sort.log 2>&1
timeout 300 python scripts/debug_c1.py > gpurun_out/debug_c1.log 2>&1
timeout 600 python scripts/power_exp.py C4 3 > gpurun_out/power_exp_c4.log 2>&1
timeout 300 python scripts/power_exp.py C3 4 > gpurun_out/power_exp_c3.log 2>&1
timeout 300 python scripts/power_exp.py C2 50 > gpurun_out/power_exp_c2.log 2>&1
