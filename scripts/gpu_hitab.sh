#!/bin/bash
# Hit-path attribution at C3 (rank 0 of 8 shard), alternating launches:
# product / sign test only (2048) / meta-only pushes / hit warps skip / both / no epilogue.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
AB_SHARD=0/8 timeout 900 python scripts/ab_env.py C3 6 "X=0" "F=2048" "F=2097152" "F=4194304" "F=6291456" "F=256" > gpurun_out/hitab.txt 2>&1
AB_SHARD=0/8 timeout 900 python scripts/ab_env.py C3 6 "X=0" "FASTED_RES_HIT=0" "F=2048,FASTED_RES_HIT=0" >> gpurun_out/hitab.txt 2>&1
