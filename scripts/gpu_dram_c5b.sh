#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for H in 1 2; do
FASTED_L2_HINT=$H timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:join_tc_mc -s 1 -c 1 --csv --log-file gpurun_out/dram_c5_H$H.csv python scripts/ncu_join.py C5 75776 0 7.2300123612099165 > gpurun_out/dram_c5_H$H.log 2>&1
done
