#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
FASTED_RES_HIT=2 FASTED_MC_HIT=2 FASTED_STREAM_HIT=2 timeout 600 python scripts/check_flag.py 33554432 > gpurun_out/pack_check.txt 2>&1
AB_SHARD=0/8 timeout 900 python scripts/ab_env.py C3 8 "X=0" "F=33554432" > gpurun_out/pack_ab.txt 2>&1
FASTED_RES_HIT=2 timeout 300 python scripts/trace_res.py C3 75776 0,33554432 > gpurun_out/pack_trace.txt 2>&1
