"""GPU FP64 truth and pair accuracy vs FP64 (the paper's Eq. 3 / Table 6),
pinned to the reference's own numbers.  Run with -m gpu."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

import paper_2508_21230_b200 as F  # noqa: E402
from paper_2508_21230_b200 import accuracy, engine  # noqa: E402


def _numpy_fp64_pairs(x, rows, eps):
    """oracle.py:26-64 restated (pairwise_sqdist_fp64 + sqrt threshold)."""
    d2 = F.pairwise_sqdist_fp64(x, rows)
    keep = np.sqrt(d2) <= eps
    rr, cc = np.nonzero(keep)
    i, j, d = (rows[rr] + 1).astype(np.uint32), (cc + 1).astype(np.uint32), d2[rr, cc]
    o = np.lexsort((j, i))
    return i[o], j[o], d[o]


@pytest.mark.parametrize("n,d,eps", [(700, 45, 2.2), (1000, 300, 7.0), (257, 16, 0.9)])
def test_fp64_rows_bit_exact_vs_numpy(n, d, eps):
    x = F.synthetic_rows(100000, d, 7, 0, n)
    rows = np.array([0, 5, 77, n - 1, n // 2], dtype=np.int64)
    gi, gj, gd = accuracy.fp64_truth_rows(x, rows, eps)
    ni, nj, nd = _numpy_fp64_pairs(x, rows, eps)
    assert np.array_equal(gi, ni) and np.array_equal(gj, nj)
    assert np.array_equal(gd.view(np.uint64), nd.view(np.uint64))


def test_c1_accuracy_matches_reference(golden_meta):
    """Exact kernel (== reference bits) against the GPU FP64 truth over ALL
    C1 points reproduces the reference's own overlap_accuracy; the tcgen05
    path is at least as accurate."""
    c1 = golden_meta["C1"]
    ref = golden_meta.get("C1_accuracy")
    ds = F.generate_synthetic(c1["n"], c1["d"], seed=c1["seed"])
    hd = F.to_half(ds)
    rows = np.arange(c1["n"], dtype=np.int64)
    ex = F.self_join(hd, c1["epsilon"], mode="exact")
    acc_ex = accuracy.accuracy_vs_fp64(ds.values, ex, c1["epsilon"], rows)
    tc = F.self_join(hd, c1["epsilon"])
    acc_tc = accuracy.accuracy_vs_fp64(ds.values, tc, c1["epsilon"], rows)
    print("C1 accuracy exact:", acc_ex, "tc:", acc_tc, "reference:", ref)
    if ref is not None:
        assert acc_ex["truth_pairs"] == ref["truth_pairs"]
        assert abs(acc_ex["overlap"] - ref["overlap"]) < 1e-12
        assert abs(acc_ex["err_mean"] - ref["err_mean"]) < 1e-12
    assert acc_tc["overlap"] >= acc_ex["overlap"] - 1e-4


def test_row_block_accuracy_helper():
    ds = F.generate_synthetic(5000, 64, seed=2)
    hd = F.to_half(ds)
    dd = engine.upload(hd, 0)
    rows = accuracy.sample_row_blocks(ds.n, blocks=3, seed=1)
    part = accuracy.join_row_blocks(dd, 2.6, rows)
    full = F.self_join(hd, 2.6)
    keep = np.isin(full.i.astype(np.int64) - 1, rows)
    assert np.array_equal(part.i, full.i[keep]) and np.array_equal(part.j, full.j[keep])
    acc = accuracy.accuracy_vs_fp64(ds.values, part, 2.6, rows)
    assert 0.98 <= acc["overlap"] <= 1.0 and acc["sample_points"] == len(rows)
