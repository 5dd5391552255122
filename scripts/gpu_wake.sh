#!/bin/bash
# Does the epilogue's accumulator wake-up limit C3 (with spin MMA waits + pacing)?
# product vs epilogue spin, and the no-epilogue ceiling with / without epilogue spin.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python scripts/ab_env.py C3 4 "X=0" "F=134217728" "F=256" "F=134217984" >> gpurun_out/wake_ab.txt 2>&1
FASTED_RES_HIT=2 timeout 300 python scripts/trace_res.py C3 75776 256 > gpurun_out/wake_trace.txt 2>&1
FASTED_RES_HIT=2 timeout 300 python scripts/trace_res.py C3 75776 134217984 >> gpurun_out/wake_trace.txt 2>&1
