#!/bin/bash
# Round-2 final evidence: GPU suite, smoke, bench (+ reference arm), one full C4 launch and a
# --set full C4 slice under ncu, the bench command's launch list.
cd "$(dirname "$0")/.."
bash scripts/gpu_r2.sh
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,lts__t_sector_hit_rate.pct,sm__cycles_elapsed.avg.per_second
timeout 900 ncu --metrics $M --clock-control none -k regex:join_tc_kernel -s 2 -c 1 --csv --log-file gpurun_out/fin_c4_fulllaunch.csv python scripts/ncu_join.py C4 1000064 40 > gpurun_out/fin_c4_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:join_tc_kernel -s 2 -c 1 -o gpurun_out/fin_c4_slice python scripts/ncu_join.py C4 131072 40 > gpurun_out/fin_c4_slice.log 2>&1
ncu -i gpurun_out/fin_c4_slice.ncu-rep --page details > gpurun_out/fin_c4_slice_details.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/fin_launches_c4.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-accuracy --no-symmetric --no-configs --e2e-steps 1 > gpurun_out/fin_launches.log 2>&1
