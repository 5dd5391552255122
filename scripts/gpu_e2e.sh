#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python scripts/e2e_breakdown.py C4 > gpurun_out/e2e_breakdown.log 2>&1
