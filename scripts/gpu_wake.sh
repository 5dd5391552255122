#!/bin/bash
# MMA-warp wake-up after the accumulator release, hit-warp kernel: suspend vs spin waits.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
FASTED_RES_HIT=2 timeout 300 python scripts/trace_res.py C3 75776 256,8448,0,8192 > gpurun_out/wake_trace.txt 2>&1
FASTED_RES_HIT=0 timeout 300 python scripts/trace_res.py C3 75776 256,8448 >> gpurun_out/wake_trace.txt 2>&1
