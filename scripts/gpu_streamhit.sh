#!/bin/bash
# CTA-pair streaming kernel: hit warps (FASTED_STREAM_HIT=2) vs not; C4 and a C5 S~64 shard.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
out=gpurun_out/streamhit.txt
: > $out
timeout 900 python -m pytest tests/test_gpu.py -x -q -k "cta_pair or multicast" 2>&1 | tail -2 >> $out
python scripts/ab_env.py C4 4 FASTED_STREAM_HIT=0 FASTED_STREAM_HIT=2 2>&1 | tail -2 >> $out
AB_SHARD=0/8 AB_EPS=6.97276473038035 python scripts/ab_env.py C5 4 FASTED_STREAM_HIT=0 FASTED_STREAM_HIT=2 2>&1 | tail -2 >> $out
cat $out
