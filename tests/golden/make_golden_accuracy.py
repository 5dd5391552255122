"""Reference accuracy known answer at C1 (run once, dev container only):
overlap_accuracy / distance_error_stats of the reference's mixed join
against its own brute_force_fp64 (analysis.py:127-219, oracle.py:43-64).

    NUMBA_CACHE_DIR=/tmp/nb python tests/golden/make_golden_accuracy.py
"""
import json
import os
import sys
import time

sys.path.insert(0, "/root/reference/pkg/src")
import mpjoin  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
t0 = time.time()
ds = mpjoin.generate_synthetic(16384, 128, seed=12345)
eps = 3.973260466174982
rs = mpjoin.self_join(mpjoin.to_half(ds), eps, mpjoin.TileConfig(workers=8))
truth = mpjoin.brute_force_fp64(ds, eps)
ov = mpjoin.overlap_accuracy(rs, truth)
st = mpjoin.distance_error_stats(rs, truth)
rec = {"n": 16384, "d": 128, "seed": 12345, "epsilon": eps, "overlap": ov,
       "err_mean": st.err_mean, "err_std": st.err_std, "matched_pairs": st.matched_pairs,
       "truth_pairs": len(truth), "mixed_pairs": len(rs), "seconds": time.time() - t0}
path = os.path.join(HERE, "reference_meta.json")
meta = json.load(open(path))
meta["C1_accuracy"] = rec
with open(path, "w") as f:
    json.dump(meta, f, indent=1, sort_keys=True)
    f.write("\n")
print(rec)
