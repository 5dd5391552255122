#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu.py -m gpu -q -x -k "hit or resident or multicast or sparse or pipeline or symmetric or golden" > gpurun_out/hq4_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/hq4_pytest.log
for r in 1 2 3; do
for lib in paper_2508_21230_b200/libfasted_exp_prev.so paper_2508_21230_b200/libfasted_exp.so; do
  echo "== $lib" >> gpurun_out/hq4_ab.txt
  FASTED_LIB=$lib AB_SHARD=0/8 timeout 600 python scripts/ab_env.py C3 5 "X=0" >> gpurun_out/hq4_ab.txt 2>&1
done
done
FASTED_RES_HIT=2 timeout 300 python scripts/trace_res.py C3 75776 0 > gpurun_out/hq4_trace.txt 2>&1
