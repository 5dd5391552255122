#!/bin/bash
# A/B: ring hand-off (FASTED_RES_HIT=18) vs shared queue (product, 2 hit warps), C3 full;
# and HBM bytes of one C3 launch per variant (product, ring, NOEPI) under ncu.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python scripts/ab_env.py C3 4 "X=0" "FASTED_RES_HIT=18" >> gpurun_out/ring_ab.txt 2>&1
AB_SHARD=0/8 timeout 900 python scripts/ab_env.py C3 6 "X=0" "FASTED_RES_HIT=18" >> gpurun_out/ring_ab.txt 2>&1
M=dram__bytes_read.sum,gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,lts__t_sector_hit_rate.pct
for v in "X=0:0" "FASTED_RES_HIT=18:0" "X=0:256"; do
  env=${v%%:*}; fl=${v##*:}
  env $env FASTED_LIB=paper_2508_21230_b200/libfasted_exp.so timeout 600 ncu --metrics $M --clock-control none -k regex:join_tc_res -s 1 -c 1 --csv python scripts/ncu_join.py C3 1000064 $((32 + fl)) > gpurun_out/ring_ncu_${env}_${fl}.csv 2>&1
done
