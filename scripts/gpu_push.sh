#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
FASTED_RES_HIT=2 timeout 300 python scripts/trace_res.py C3 75776 0 > gpurun_out/push_trace.txt 2>&1
