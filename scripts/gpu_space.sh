#!/bin/bash
# A/B: pacing of the streaming CTA-pair kernel (C4), FASTED_STREAM_PACE_W blocks of 64 tile layers.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1200 python scripts/ab_env.py C4 4 "FASTED_STREAM_PACE_W=0" "FASTED_STREAM_PACE_W=1" "FASTED_STREAM_PACE_W=4" "FASTED_STREAM_PACE_W=16" >> gpurun_out/space_ab.txt 2>&1
M=dram__bytes_read.sum,gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,lts__t_sector_hit_rate.pct,sm__cycles_elapsed.avg.per_second
for w in 0 1 4; do
  FASTED_STREAM_PACE_W=$w FASTED_LIB=paper_2508_21230_b200/libfasted_exp.so timeout 900 ncu --metrics $M --clock-control none -k regex:join_tc_kernel -s 2 -c 1 --csv python scripts/ncu_join.py C4 1000064 40 > gpurun_out/space_ncu_w$w.csv 2>&1
done
