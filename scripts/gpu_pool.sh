#!/bin/bash
# Default mempool release threshold (FASTED_POOL_KEEP=1: keep 1 GiB) vs driver default (0), C2, alternating processes.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for r in 1 2 3; do
for k in 0 1; do
  echo "== FASTED_POOL_KEEP=$k" >> gpurun_out/pool_ab.txt
  FASTED_POOL_KEEP=$k timeout 600 python scripts/ab_env.py C2 100 "X=0" 2>&1 | cut -c1-100 >> gpurun_out/pool_ab.txt
done
done
