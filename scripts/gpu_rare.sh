#!/bin/bash
# Dense-output rare path A/B (staged writers, no hit warps): hybrid (product), always
# transposed rows (RARE_ROWS), always per-lane masks (RARE_LM); C5 shard S~4096 / S~1024, C2.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
AB_EPS=7.2300123612099165 AB_SHARD=0/8 timeout 900 python scripts/ab_env.py C5 2 "X=0" "F=262144" "F=131072" >> gpurun_out/rare_ab.txt 2>&1
AB_EPS=7.1352369182727085 AB_SHARD=0/8 timeout 900 python scripts/ab_env.py C5 2 "X=0" "F=262144" "F=131072" >> gpurun_out/rare_ab.txt 2>&1
timeout 600 python scripts/ab_env.py C2 30 "X=0" "F=262144" "F=131072" >> gpurun_out/rare_ab.txt 2>&1
