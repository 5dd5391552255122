#!/bin/bash
# C3 per-launch time across this round's commits (product builds from each commit's sources).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
P=paper_2508_21230_b200
for r in 1 2; do
for lib in libfasted_r1 libfasted_bis_4fb0667 libfasted_bis_2f4d6fc libfasted_bis_a36774c libfasted_bis_dd368f5 libfasted_bis_3e9ec37 libfasted; do
  echo "== $lib" >> gpurun_out/bisect.txt
  FASTED_LIB=$P/$lib.so AB_SHARD=0/8 timeout 600 python scripts/ab_env.py C3 6 "X=0" >> gpurun_out/bisect.txt 2>&1
done
done
