#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python scripts/e2e_trace.py C4 > gpurun_out/e2e_trace.log 2>&1
