"""Kernel form for the column-segment launches of upload_segmented's first
row chunk (C4: rows [0, 250112) x a 62.5K-column segment): CTA-pair
(FASTED_JOIN_LOW_OUTPUT, forced with FASTED_CTA_GROUP=2) vs the default
selection, ms per launch and TFLOPS.
usage: python scripts/seg_forms.py"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2508_21230_b200 as F  # noqa: E402
from bench import SEED, WORKLOADS  # noqa: E402
from paper_2508_21230_b200 import _lib, engine  # noqa: E402
# env knobs and diagnostic flags exist only in the experiment build
_lib.LIB_PATH = os.path.abspath(os.environ.get("FASTED_LIB", _lib.EXP_LIB_PATH))

name, n, d, eps = WORKLOADS["C4"]
hd = F.to_half(F.generate_synthetic(n, d, seed=SEED))
dd = engine.upload(hd, 0)
es = float(np.float32(np.float32(eps) ** 2))
L = _lib.load()
cnt = torch.zeros(2, dtype=torch.int64, device="cuda")
rec = torch.empty((4_000_000, 4), dtype=torch.int32, device="cuda")
s = torch.cuda.current_stream()
rows = (0, 250112)
for cols in ((312448, 374912), (0, 312448)):
    for label, env in (("default", "0"), ("pair", "2")):
        os.environ["FASTED_CTA_GROUP"] = env
        flags = _lib.JOIN_TC | _lib.JOIN_LOW_OUTPUT
        engine.join_raw(dd, es, flags, rows, cols, rec, rec.shape[0], cnt, s.cuda_stream)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(3):
            engine.join_raw(dd, es, flags, rows, cols, rec, rec.shape[0], cnt, s.cuda_stream)
        e1.record(s)
        e1.synchronize()
        ms = e0.elapsed_time(e1) / 3
        fl = 2.0 * (rows[1] - rows[0]) * (cols[1] - cols[0]) * d
        kern = L.fasted_join_kernel_name(dd.d_pad, rows[1] - rows[0], cols[1] - cols[0],
                                         flags).decode()
        print(f"rows {rows} cols {cols} {label:8s} {kern:36s} {ms:8.2f} ms "
              f"{fl / ms / 1e9:7.1f} TFLOPS count {int(cnt[0])}", flush=True)
os.environ.pop("FASTED_CTA_GROUP", None)
