#!/bin/bash
# A/B: hit-queue hand-off by st.async + complete_tx (default) vs generic
# shared stores + release arrive (FASTED_JOIN_DIAG_GENERICQ), C3 shard 0/8;
# push-phase traces with the slot-wait stamp (libfasted_exp_slot.so).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for r in 1 2 3; do
AB_SHARD=0/8 timeout 600 python scripts/ab_env.py C3 6 "X=0" "F=67108864" >> gpurun_out/genq_ab.txt 2>&1
done
for f in 0 67108864; do
TRACE_SLOT=1 FASTED_LIB=paper_2508_21230_b200/libfasted_exp_slot.so FASTED_RES_HIT=2 timeout 300 python scripts/trace_res.py C3 75776 $f >> gpurun_out/genq_trace.txt 2>&1
done
