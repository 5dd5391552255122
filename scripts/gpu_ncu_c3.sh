#!/bin/bash
# ncu --set full (source-level stall reasons) of one C3 shard launch of the
# product kernel (join_tc_res_kernel<2> + 2 hit warps, FASTED_JOIN_SPARSE).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:join_tc_res -s 1 -c 1 \
  -o gpurun_out/ncu_c3_res python scripts/ncu_join.py C3 75776 32 > gpurun_out/ncu_c3_res.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_c3_res.log
