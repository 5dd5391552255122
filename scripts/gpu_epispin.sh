#!/bin/bash
# A/B: epilogue accumulator wait by try_wait suspend (product) vs test_wait spin
# (FASTED_JOIN_DIAG_EPISPIN), with the MMA/producer spin default in both.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python scripts/ab_env.py C4 4 "X=0" "F=134217728" >> gpurun_out/epispin_ab.txt 2>&1
timeout 600 python scripts/ab_env.py C3 4 "X=0" "F=134217728" >> gpurun_out/epispin_ab.txt 2>&1
AB_EPS=7.049487707996186 AB_SHARD=0/8 timeout 900 python scripts/ab_env.py C5 2 "X=0" "F=134217728" >> gpurun_out/epispin_ab.txt 2>&1
AB_EPS=7.2300123612099165 AB_SHARD=0/8 timeout 900 python scripts/ab_env.py C5 2 "X=0" "F=134217728" >> gpurun_out/epispin_ab.txt 2>&1
timeout 600 python scripts/ab_env.py C2 30 "X=0" "F=134217728" >> gpurun_out/epispin_ab.txt 2>&1
