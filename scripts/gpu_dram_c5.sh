#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for F in 0 2; do
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:join_tc_mc -s 1 -c 1 --csv --log-file gpurun_out/dram_c5_F$F.csv python scripts/ncu_join.py C5 75776 $F 7.2300123612099165 > gpurun_out/dram_c5_F$F.log 2>&1
done
