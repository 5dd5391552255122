#!/bin/bash
# Multicast kernel: hit warps (FASTED_MC_HIT=2) vs epilogue warps; tests, C2, C5 shard S~4096 / S~256.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
out=gpurun_out/ab_mchit.txt
: > $out
timeout 900 python -m pytest tests/test_gpu.py -x -q -k "multicast or resident" 2>&1 | tail -2 >> $out
python scripts/ab_env.py C2 30 FASTED_MC_HIT=0 FASTED_MC_HIT=2 2>&1 | tail -2 >> $out
AB_SHARD=0/8 AB_EPS=7.2300123612099165 python scripts/ab_env.py C5 4 FASTED_MC_HIT=0 FASTED_MC_HIT=2 2>&1 | tail -2 >> $out
AB_SHARD=0/8 AB_EPS=7.049487707996186 python scripts/ab_env.py C5 4 FASTED_MC_HIT=0 FASTED_MC_HIT=2 2>&1 | tail -2 >> $out
cat $out
