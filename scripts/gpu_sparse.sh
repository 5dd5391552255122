#!/bin/bash
# FASTED_JOIN_SPARSE hint: GPU suite, C3 / C5 S~256 A/B (hit warps on/off by env override).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
out=gpurun_out/sparse.txt
: > $out
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_sparse.log 2>&1; tail -2 gpurun_out/pytest_sparse.log >> $out
python scripts/ab_env.py C3 8 FASTED_RES_HIT=0 FASTED_RES_HIT=2 2>&1 | tail -2 >> $out
AB_SHARD=0/8 AB_EPS=7.049487707996186 python scripts/ab_env.py C5 4 FASTED_MC_HIT=0 FASTED_MC_HIT=2 2>&1 | tail -2 >> $out
python -c "
import sys; sys.path.insert(0,'.')
from paper_2508_21230_b200 import _lib, engine
L=_lib.load()
for d,r,c,pairs in ((128,1000064,1000064,74552502),(960,1000064,1000064,49048308),(512,60032,60032,3623702)):
    f=engine.form_hints(pairs,(0,r),(0,c)); print(d, f, L.fasted_join_kernel_name(d,r,c,f).decode())
" >> $out 2>&1
cat $out
