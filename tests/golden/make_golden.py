"""Generate golden vectors by running the REFERENCE package itself.

Run in the dev container only (needs /root/reference and numba):

    NUMBA_CACHE_DIR=/tmp/nb python tests/golden/make_golden.py [--big]

Outputs (committed; small):
  tests/golden/reference_cases.npz   reference to_half + self_join on small
                                      datasets (and one compute_block_tile)
  tests/golden/reference_meta.json    error messages, C1 known answer,
                                      sampled-tile pairs for the C2-C5 shapes

Every array is the reference's own output (mpjoin.to_half / self_join /
compute_block_tile / brute_force_fp64); nothing here comes from this repo's
oracle or kernels.  tests/test_oracle.py pins the oracle to these files and
the GPU tests compare the CUDA path against them.
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import mpjoin  # noqa: E402
from mpjoin import cli as mcli  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))

# (name, n, d, seed, lo, hi, epsilon)
SYNTHETIC = [
    ("uniform_700x45", 700, 45, 3, 0.0, 1.0, 2.2),
    ("spec_512x128", 512, 128, 12345, 0.0, 1.0, 4.3),      # SPEC.md:525 criterion 3 shape
    ("ragged_130x17", 130, 17, 9, -3.0, 5.0, 9.0),         # n and d both padded
    ("wide_300x64", 300, 64, 21, -500.0, 500.0, 3200.0),   # large magnitudes
    ("c1_slice_1024x128", 1024, 128, 12345, 0.0, 1.0, 3.973260466174982),
]

# Sampled 128x128 tiles of the headline shapes.
# (name, n, d, eps, [(row_block, col_block), ...])
SAMPLED = [
    ("C2", 60000, 512, 8.48414709018062, [(0, 0), (3, 200), (468, 468), (468, 5)]),
    ("C3", 1000000, 128, 3.685431479161428, [(0, 0), (4000, 17), (7812, 7812), (7812, 3)]),
    ("C4", 1000000, 960, 11.700486640655093, [(0, 0), (1234, 4321), (7812, 7812)]),
    ("C5", 5000000, 384, 7.1352369182727085, [(0, 0), (39062, 39062), (20000, 7)]),
]


def rs_arrays(rs):
    return rs.i.astype(np.uint32), rs.j.astype(np.uint32), rs.dist_sq.astype(np.float32)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--big", action="store_true", help="also the C1 full join and C2-C5 tiles")
    args = ap.parse_args()
    out = {}
    meta = {"reference": "mpjoin " + mpjoin.__version__, "cases": {}}

    # to_half known answers (test_dataset.py:130-139 style) incl. subnormals/ties
    vals = np.array([[0.1, 1.0, -2.5, 65504.0, 65519.0, 6.0e-8, 2.9802322e-08,
                      5.96e-08, -1e-9, 3.0e-5, 0.33333334, 1024.5, 2049.0, 2051.0]],
                    np.float32)
    hd = mpjoin.to_half(mpjoin.Dataset(vals))
    out["tohalf_in"] = vals
    out["tohalf_values"] = hd.values.view(np.uint16)
    out["tohalf_norms"] = hd.norms
    try:
        mpjoin.to_half(mpjoin.Dataset(np.array([[1.0, 2.0], [3.0, 70000.0]], np.float32)))
    except mpjoin.RangeError as exc:
        meta["range_error_message"] = str(exc)
    try:
        mpjoin.to_half(mpjoin.Dataset(np.array([[65520.0]], np.float32)))
    except mpjoin.RangeError as exc:
        meta["range_error_message_65520"] = str(exc)

    for name, n, d, seed, lo, hi, eps in SYNTHETIC:
        ds = mpjoin.generate_synthetic(n, d, seed=seed, lo=lo, hi=hi)
        hd = mpjoin.to_half(ds)
        rs = mpjoin.self_join(hd, eps, mpjoin.TileConfig(workers=8))
        i, j, dd = rs_arrays(rs)
        out[f"{name}_x"] = ds.values
        out[f"{name}_values"] = hd.values.view(np.uint16)
        out[f"{name}_norms"] = hd.norms
        out[f"{name}_i"], out[f"{name}_j"], out[f"{name}_d"] = i, j, dd
        meta["cases"][name] = {
            "n": n, "d": d, "seed": seed, "lo": lo, "hi": hi, "epsilon": eps,
            "pairs": len(rs), "selectivity": mpjoin.selectivity(rs),
            "result_sha256": hashlib.sha256(mcli.pairs_payload(rs)).hexdigest(),
            "dataset_sha256": mcli.dataset_sha256(ds),
        }
        print(name, len(rs), mpjoin.selectivity(rs))

    # integer regime: mixed == FP64 (criterion 4)
    rng = np.random.default_rng(4)
    xi = rng.integers(-8, 9, size=(200, 16)).astype(np.float32)
    ds = mpjoin.Dataset(xi)
    hd = mpjoin.to_half(ds)
    rs = mpjoin.self_join(hd, 6.0)
    truth = mpjoin.brute_force_fp64(ds, 6.0)
    assert rs.same_pairs(truth)
    out["integer_x"] = xi
    out["integer_i"], out["integer_j"], out["integer_d"] = rs_arrays(rs)
    meta["cases"]["integer"] = {"epsilon": 6.0, "pairs": len(rs)}

    # hand fixtures
    tri = mpjoin.to_half(mpjoin.Dataset(np.array([[0.0, 0.0], [3.0, 4.0]], np.float32)))
    out["tri_i"], out["tri_j"], out["tri_d"] = rs_arrays(mpjoin.self_join(tri, 5.0))
    same = mpjoin.to_half(mpjoin.Dataset(np.ones((3, 4), np.float32) * 0.7))
    rs = mpjoin.self_join(same, 0.5)
    meta["cases"]["three_identical"] = {"pairs": len(rs), "selectivity": mpjoin.selectivity(rs)}
    out["same_i"], out["same_j"], out["same_d"] = rs_arrays(rs)
    # duplicates at eps = 0: the reference keeps every exact-duplicate pair
    base = mpjoin.generate_synthetic(50, 24, seed=8).values
    dup = np.concatenate([base, base[::7]])
    hdd = mpjoin.to_half(mpjoin.Dataset(dup))
    out["dup_x"] = dup
    out["dup_i"], out["dup_j"], out["dup_d"] = rs_arrays(mpjoin.self_join(hdd, 0.0))

    # one compute_block_tile (tiling.py:199) off the diagonal
    ds = mpjoin.generate_synthetic(384, 64, seed=31)
    hd = mpjoin.to_half(ds)
    es = np.float32(np.float32(3.3) * np.float32(3.3))
    ti, tj, td = mpjoin.compute_block_tile(hd, mpjoin.TileCoord(2, 1), es, mpjoin.TileConfig())
    out["tile_x"] = ds.values
    out["tile_i"], out["tile_j"], out["tile_d"] = ti, tj, td

    # fvecs known answer
    meta["fvecs_example"] = "see tests/test_host.py (format from dataset.py:89-132)"

    if args.big:
        t0 = time.time()
        ds = mpjoin.generate_synthetic(16384, 128, seed=12345)
        hd = mpjoin.to_half(ds)
        st = mpjoin.EngineStats()
        rs = mpjoin.self_join(hd, 3.973260466174982, mpjoin.TileConfig(workers=8), stats_out=st)
        meta["C1"] = {
            "n": 16384, "d": 128, "seed": 12345, "epsilon": 3.973260466174982,
            "pairs": len(rs), "selectivity": mpjoin.selectivity(rs),
            "result_sha256": hashlib.sha256(mcli.pairs_payload(rs)).hexdigest(),
            "dataset_sha256": mcli.dataset_sha256(ds),
            "reference_kernel_seconds_8_workers_dev_container": st.kernel_wall_seconds,
        }
        print("C1", meta["C1"], time.time() - t0)
        meta["sampled_tiles"] = {}
        for name, n, d, eps, tiles in SAMPLED:
            t0 = time.time()
            ds = mpjoin.generate_synthetic(n, d, seed=12345)
            hd = mpjoin.to_half(ds)
            es = np.float32(np.float32(eps) * np.float32(eps))
            rec = {"n": n, "d": d, "seed": 12345, "epsilon": eps, "tiles": []}
            for (rb, cb) in tiles:
                ti, tj, td = mpjoin.compute_block_tile(hd, mpjoin.TileCoord(rb, cb), es,
                                                       mpjoin.TileConfig())
                key = f"{name}_{rb}_{cb}"
                out[key + "_i"], out[key + "_j"], out[key + "_d"] = ti, tj, td
                out[key + "_rownorms"] = hd.norms[rb * 128:(rb + 1) * 128]
                out[key + "_colnorms"] = hd.norms[cb * 128:(cb + 1) * 128]
                rec["tiles"].append({"row_block": rb, "col_block": cb, "pairs": int(len(ti))})
            meta["sampled_tiles"][name] = rec
            print(name, rec, time.time() - t0)
            del ds, hd

    np.savez_compressed(os.path.join(HERE, "reference_cases.npz"), **out)
    with open(os.path.join(HERE, "reference_meta.json"), "w") as f:
        json.dump(meta, f, indent=1, sort_keys=True)
        f.write("\n")


if __name__ == "__main__":
    main()
