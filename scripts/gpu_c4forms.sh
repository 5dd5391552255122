#!/bin/bash
# C4 streaming pair with pacing: hit warps (product, SPARSE hint) vs none; 16 vs 8 epilogue warps.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1500 python scripts/ab_env.py C4 3 "X=0" "FASTED_STREAM_HIT=0" "FASTED_STREAM_EPI=8,FASTED_STREAM_HIT=0" >> gpurun_out/c4forms_ab.txt 2>&1
