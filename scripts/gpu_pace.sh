#!/bin/bash
# A/B: resident-kernel pacing (bounded drift between co-running pairs, FASTED_PACE_W layers).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python scripts/ab_env.py C3 3 "FASTED_PACE_W=0" "FASTED_PACE_W=2" "FASTED_PACE_W=4" "FASTED_PACE_W=8" >> gpurun_out/pace_ab.txt 2>&1
M=dram__bytes_read.sum,gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,lts__t_sector_hit_rate.pct
for w in 0 2 4; do
  FASTED_PACE_W=$w FASTED_LIB=paper_2508_21230_b200/libfasted_exp.so timeout 600 ncu --metrics $M --clock-control none -k regex:join_tc_res -s 1 -c 1 --csv python scripts/ncu_join.py C3 1000064 32 > gpurun_out/pace_ncu_c3_w$w.csv 2>&1
done
AB_EPS=7.049487707996186 AB_SHARD=0/8 timeout 900 python scripts/ab_env.py C5 2 "FASTED_PACE_W=0" "FASTED_PACE_W=2" "FASTED_PACE_W=4" >> gpurun_out/pace_ab.txt 2>&1
AB_EPS=7.2300123612099165 AB_SHARD=0/8 timeout 900 python scripts/ab_env.py C5 2 "FASTED_PACE_W=0" "FASTED_PACE_W=2" "FASTED_PACE_W=4" >> gpurun_out/pace_ab.txt 2>&1
timeout 600 python scripts/ab_env.py C2 20 "FASTED_PACE_W=0" "FASTED_PACE_W=2" "FASTED_PACE_W=4" >> gpurun_out/pace_ab.txt 2>&1
