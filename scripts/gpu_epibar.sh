#!/bin/bash
# Epilogue accumulator wait through one waiter + a named barrier (FASTED_JOIN_DIAG_EPIBAR).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python scripts/ab_env.py C3 4 "X=0" "F=268435456" >> gpurun_out/epibar_ab.txt 2>&1
AB_SHARD=0/8 timeout 900 python scripts/ab_env.py C3 8 "X=0" "F=268435456" >> gpurun_out/epibar_ab.txt 2>&1
AB_EPS=7.049487707996186 AB_SHARD=0/8 timeout 900 python scripts/ab_env.py C5 2 "X=0" "F=268435456" >> gpurun_out/epibar_ab.txt 2>&1
