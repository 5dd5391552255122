#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for F in 8 65544; do
timeout 900 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:join_tc_kernel -s 2 -c 1 --csv --log-file gpurun_out/bpf_$F.csv python scripts/ncu_join.py C4 131072 $F > gpurun_out/bpf_$F.log 2>&1
done
timeout 1500 python scripts/tune.py C4 2 "CG=2,G=16384" "CG=2,G=16384,F=65536" "CG=2,G=16384" "CG=2,G=16384,F=65536" > gpurun_out/tune_c4_bpf.log 2>&1
