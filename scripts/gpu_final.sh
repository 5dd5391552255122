#!/bin/bash
# Round evidence for the committed state: full GPU suite (incl. full-size parity), smoke,
# default bench line, ncu launch list of the bench command, ncu --set full of a C4 slice.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_final.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_final.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_final.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_final.log
timeout 1200 python bench.py > gpurun_out/bench_final.log 2>&1; echo "rc=$?" >> gpurun_out/bench_final.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_final.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-accuracy --no-symmetric --e2e-steps 1 > gpurun_out/launches_final.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:join_tc_kernel -s 2 -c 1 -o gpurun_out/ncu_c4_final python scripts/ncu_join.py C4 131072 40 > gpurun_out/ncu_c4_final.log 2>&1
