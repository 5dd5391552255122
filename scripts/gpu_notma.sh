#!/bin/bash
# C3 mainloop attribution (rank 0 of 8): no epilogue / no epilogue + no TMA / TMA alone,
# and the sort after the evict_first stream loads + register-cached rank sort.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
AB_SHARD=0/8 timeout 900 python scripts/ab_env.py C3 6 "X=0" "F=256" "F=8388864" "F=768" > gpurun_out/notma.txt 2>&1
FASTED_RES_HIT=2 timeout 300 python scripts/trace_res.py C3 75776 8388864 > gpurun_out/notma_trace.txt 2>&1
timeout 600 python -m pytest tests/test_gpu.py -m gpu -q -x -k "sort or long_rows or pipeline" > gpurun_out/notma_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/notma_pytest.log
bash scripts/gpu_sort_prof.sh
