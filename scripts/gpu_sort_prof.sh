#!/bin/bash
# Launch list of the sort kernels at C5 S4096 (one rank of 8): per-kernel time.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:"hist|scatter|rank_rows|bucket_rows|short_rows|scan_|long_rows" --csv \
  --log-file gpurun_out/sort_launches_s4096.csv \
  python scripts/c5_sweep.py --shard 0/8 --reps 1 --only S4096 > gpurun_out/sort_prof.log 2>&1; echo "rc=$?" >> gpurun_out/sort_prof.log
