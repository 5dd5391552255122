#!/bin/bash
# st.async hit-queue hand-off: GPU suite, racecheck over every form, hit-warp trace at C3,
# A/B of the product C3/C5 kernels against the previous build (libfasted_exp_prev.so).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/hq_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/hq_pytest.log
FASTED_RES_HIT=2 timeout 300 python scripts/trace_res.py C3 75776 0,256 > gpurun_out/hq_trace.txt 2>&1
for lib in paper_2508_21230_b200/libfasted_exp_prev.so paper_2508_21230_b200/libfasted_exp.so; do
  echo "== $lib" >> gpurun_out/hq_ab.txt
  FASTED_LIB=$lib AB_SHARD=0/8 timeout 600 python scripts/ab_env.py C3 5 "X=0" >> gpurun_out/hq_ab.txt 2>&1
done
bash scripts/gpu_sanitize.sh > /dev/null 2>&1
