#!/bin/bash
# A/B: epilogue accumulator wait by try_wait suspend (0) vs test_wait + nanosleep backoff.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for r in 1 2; do
AB_SHARD=0/8 timeout 600 python scripts/ab_env.py C3 6 "FASTED_EPI_SLEEP_NS=0" "FASTED_EPI_SLEEP_NS=20" "FASTED_EPI_SLEEP_NS=60" "FASTED_EPI_SLEEP_NS=150" "FASTED_EPI_SLEEP_NS=400" >> gpurun_out/sleep_ab.txt 2>&1
done
AB_SHARD=0/8 timeout 600 python scripts/ab_env.py C2 20 "FASTED_EPI_SLEEP_NS=0" "FASTED_EPI_SLEEP_NS=60" "FASTED_EPI_SLEEP_NS=150" >> gpurun_out/sleep_ab.txt 2>&1
FASTED_EPI_SLEEP_NS=60 FASTED_RES_HIT=2 timeout 300 python scripts/trace_res.py C3 75776 0 > gpurun_out/sleep_trace.txt 2>&1
