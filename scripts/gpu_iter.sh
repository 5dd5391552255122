#!/bin/bash
# Iteration check: a subset of the GPU suite (PYTEST_K), then the C5 S4096 /
# S1024 sweep rows (join + sort) and per-config kernel times (tune.py).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/it_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/it_pytest.log
for s in S4096 S1024; do
timeout 600 python scripts/c5_sweep.py --shard 0/8 --reps 2 --only $s >> gpurun_out/it_c5.jsonl 2>&1
done
timeout 600 python scripts/tune.py C3 5 "CG=0" >> gpurun_out/it_tune.log 2>&1
timeout 600 python scripts/tune.py C2 20 "CG=0" >> gpurun_out/it_tune.log 2>&1
