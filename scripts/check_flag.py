"""Bit-identity of the sorted pair set under an experiment flag (results-valid
flags only): python scripts/check_flag.py FLAG [ENV=V ...].  Runs C2 (full),
a C3 slice and a ragged case through libfasted_exp.so with and without FLAG."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_21230_b200 as F  # noqa: E402
from bench import SEED, WORKLOADS  # noqa: E402
from paper_2508_21230_b200 import _lib, engine  # noqa: E402

flag = int(sys.argv[1])
for kv in sys.argv[2:]:
    k, v = kv.split("=")
    os.environ[k] = v
X = _lib.load_experimental()
cases = [("C2", None), ("C3", (0, 65536)), ("ragged", None)]
ok = True
for name, rows in cases:
    if name == "ragged":
        n, d, eps = 9000, 136, 3.9
    else:
        _, n, d, eps = WORKLOADS[name]
    hd = F.to_half(F.generate_synthetic(n, d, seed=SEED))
    dd = engine.upload(hd, 0)
    es = float(np.float32(np.float32(eps) ** 2))
    out = []
    for fl in (0, flag):
        r = engine.join_device(dd, es, rows=rows, flags=fl, lib=X)
        out.append(engine.to_host(r))
    same = all(np.array_equal(a.view(np.uint32), b.view(np.uint32)) for a, b in zip(*out))
    print(f"{name}: pairs {len(out[0][0])} vs {len(out[1][0])}, bit-identical {same}", flush=True)
    ok &= same
print("OK" if ok else "MISMATCH")
