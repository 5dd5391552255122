#!/bin/bash
# Epilogue accumulator wait backoff re-checked under segment-major + pacing.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python scripts/ab_env.py C3 4 "FASTED_EPI_SLEEP_NS=0" "FASTED_EPI_SLEEP_NS=64" "FASTED_EPI_SLEEP_NS=200" "FASTED_EPI_SLEEP_NS=500" >> gpurun_out/sleep2_ab.txt 2>&1
AB_EPS=7.2300123612099165 AB_SHARD=0/8 timeout 900 python scripts/ab_env.py C5 2 "FASTED_EPI_SLEEP_NS=0" "FASTED_EPI_SLEEP_NS=200" >> gpurun_out/sleep2_ab.txt 2>&1
