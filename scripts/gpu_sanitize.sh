#!/bin/bash
# compute-sanitizer memcheck + racecheck over every kernel form on small
# joins: resident (d <= 256), multicast and CTA-pair streaming (d > 256),
# symmetric, exact, hit warps, and the segmented-upload pipeline (FASTED_JOIN_APPEND).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
cat > /tmp/san.py <<'PY'
import sys, os, numpy as np
sys.path.insert(0, os.getcwd())
import paper_2508_21230_b200 as F
from paper_2508_21230_b200 import _lib, engine
# the FASTED_* overrides below exist only in the experiment build
_lib.LIB_PATH = _lib.EXP_LIB_PATH
for n, d, eps in ((2000, 200, 5.4), (1500, 520, 8.6), (3000, 64, 2.6), (1500, 384, 7.7),
                  (1000, 512, 8.6)):
    hd = F.to_half(F.generate_synthetic(n, d, seed=n))
    a = F.self_join(hd, eps); b = F.self_join(hd, eps, symmetric=True)
    c = F.self_join(hd, eps, mode="exact")
    print(n, d, len(a), len(b), len(c), flush=True)
os.environ["FASTED_CTA_GROUP"] = "2"
hd = F.to_half(F.generate_synthetic(1500, 520, seed=3))
print("cg2", len(F.self_join(hd, 8.6)), flush=True)
del os.environ["FASTED_CTA_GROUP"]
# hit warps forced on (normally chosen by the FASTED_JOIN_SPARSE hint)
os.environ.update(FASTED_RES_HIT="2", FASTED_MC_HIT="2", FASTED_STREAM_HIT="2")
for n, d, eps in ((2000, 200, 5.4), (1500, 520, 8.6)):
    hd = F.to_half(F.generate_synthetic(n, d, seed=n))
    print("hit", n, d, len(F.self_join(hd, eps)), len(F.self_join(hd, eps, symmetric=True)), flush=True)
os.environ["FASTED_CTA_GROUP"] = "2"
print("hit cg2", len(F.self_join(F.to_half(F.generate_synthetic(1500, 520, seed=3)), 8.6)), flush=True)
del os.environ["FASTED_CTA_GROUP"]
for k in ("FASTED_RES_HIT", "FASTED_MC_HIT", "FASTED_STREAM_HIT"):
    del os.environ[k]
engine.SEGMENT_MIN_BYTES = 0
engine.PIPELINE_MIN_RECORDS = 0
hd = F.to_half(F.generate_synthetic(4000, 256, seed=4), pin_host=True)
hd.device_cache.clear()
print("segmented", len(F.self_join(hd, 6.0)), flush=True)
PY
timeout 1500 /usr/local/cuda/bin/compute-sanitizer --tool memcheck --print-limit 20 python /tmp/san.py > gpurun_out/sanitize_memcheck.log 2>&1; echo "rc=$?" >> gpurun_out/sanitize_memcheck.log
timeout 1500 /usr/local/cuda/bin/compute-sanitizer --tool racecheck --print-limit 20 python /tmp/san.py > gpurun_out/sanitize_racecheck.log 2>&1; echo "rc=$?" >> gpurun_out/sanitize_racecheck.log
tail -12 gpurun_out/sanitize_memcheck.log; tail -12 gpurun_out/sanitize_racecheck.log
