#!/bin/bash
# Final state (segment-major + pacing): GPU suite, smoke, bench + reference arm, one full C3
# launch under ncu, sanitizers.
cd "$(dirname "$0")/.."
bash scripts/gpu_r2.sh
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,lts__t_sector_hit_rate.pct,sm__cycles_elapsed.avg.per_second
timeout 900 ncu --metrics $M --clock-control none -k regex:join_tc_res -s 1 -c 1 --csv --log-file gpurun_out/fin2_c3_fulllaunch.csv python scripts/ncu_join.py C3 1000064 32 > gpurun_out/fin2_c3_full.log 2>&1
bash scripts/gpu_sanitize.sh > /dev/null 2>&1
