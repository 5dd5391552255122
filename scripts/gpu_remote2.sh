#!/bin/bash
# Is the accumulator-release wait (no-epilogue ceiling) set by the peer CTA's remote arrivals?
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python scripts/ab_env.py C3 4 "F=256" "F=16777472" >> gpurun_out/remote2_ab.txt 2>&1
FASTED_RES_HIT=2 timeout 300 python scripts/trace_res.py C3 75776 16777472 > gpurun_out/remote2_trace.txt 2>&1
