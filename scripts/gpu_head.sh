#!/bin/bash
# A/B: hit-queue producers read the head counter eagerly with the tail atomic (product)
# vs the per-lane lazy check (FASTED_JOIN_DIAG_HEADLAZY).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python scripts/ab_env.py C3 4 "X=0" "F=268435456" >> gpurun_out/head_ab.txt 2>&1
AB_SHARD=0/8 timeout 900 python scripts/ab_env.py C3 6 "X=0" "F=268435456" >> gpurun_out/head_ab.txt 2>&1
AB_EPS=7.049487707996186 AB_SHARD=0/8 timeout 900 python scripts/ab_env.py C5 2 "X=0" "F=268435456" >> gpurun_out/head_ab.txt 2>&1
AB_SHARD=0/8 timeout 900 python scripts/ab_env.py C4 4 "X=0" "F=268435456" >> gpurun_out/head_ab.txt 2>&1
TRACE_SLOT=1 FASTED_LIB=paper_2508_21230_b200/libfasted_exp.so FASTED_RES_HIT=2 timeout 300 python scripts/trace_res.py C3 75776 0 > gpurun_out/head_trace.txt 2>&1
