#!/bin/bash
# Evidence for the paced resident kernel: sanitizers over every kernel form, and one
# full C3 launch under ncu (HBM bytes, L2 hit rate, tensor-pipe activity).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,lts__t_sector_hit_rate.pct,sm__cycles_elapsed.avg.per_second
timeout 900 ncu --metrics $M --clock-control none -k regex:join_tc_res -s 1 -c 1 --csv --log-file gpurun_out/ev2_c3_fulllaunch.csv python scripts/ncu_join.py C3 1000064 32 > gpurun_out/ev2_c3_full.log 2>&1
bash scripts/gpu_sanitize.sh > /dev/null 2>&1
timeout 1500 /usr/local/cuda/bin/compute-sanitizer --tool synccheck --print-limit 20 python /tmp/san.py > gpurun_out/sanitize_synccheck.log 2>&1; echo "rc=$?" >> gpurun_out/sanitize_synccheck.log
