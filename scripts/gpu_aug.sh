#!/bin/bash
# Augment-step attribution at C3 (d = 128): full / no epilogue / no augment MMA /
# augment as kind::f16, alternating launches on one rank-of-8 slice; plus the
# no-epilogue trace of the MMA period.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
AB_SHARD=0/8 timeout 600 python scripts/ab_env.py C3 6 "X=0" "F=256" "F=524544" "F=1048832" "F=524288" "F=1048576" > gpurun_out/aug_ab.txt 2>&1
timeout 300 python scripts/trace_res.py C3 75776 256 > gpurun_out/aug_trace.txt 2>&1
timeout 300 python scripts/trace_res.py C3 75776 524544 >> gpurun_out/aug_trace.txt 2>&1
timeout 300 python scripts/trace_res.py C3 75776 0 >> gpurun_out/aug_trace.txt 2>&1
