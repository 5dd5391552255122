#!/bin/bash
# Round-2 check on one box: GPU parity suite (no -x: every failure listed),
# smoke(), the default bench (C4 headline + C2/C3/C5 configs), reference arm.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/r2_gpu.txt
timeout 1500 python -m pytest tests -m "gpu" -q ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/r2_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r2_smoke.log
[ -n "$NO_BENCH" ] && exit 0
timeout 1200 python bench.py > gpurun_out/r2_bench.log 2>&1; echo "rc=$?" >> gpurun_out/r2_bench.log
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2_bench_ref.log 2>&1; echo "rc=$?" >> gpurun_out/r2_bench_ref.log
