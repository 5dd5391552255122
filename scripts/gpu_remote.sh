#!/bin/bash
# Does the CTA pair's remote accumulator release set the C3 tile period?
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
AB_SHARD=0/8 timeout 900 python scripts/ab_env.py C3 6 "F=256" "F=16777472" "F=25166080" > gpurun_out/remote.txt 2>&1
FASTED_RES_HIT=2 timeout 300 python scripts/trace_res.py C3 75776 16777472 > gpurun_out/remote_trace.txt 2>&1
