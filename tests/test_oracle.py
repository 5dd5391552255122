"""Pin the CPU oracle to the reference's own outputs (tests/golden/, made by
tests/golden/make_golden.py from /root/reference).  CPU only."""

import hashlib

import numpy as np
import pytest

from paper_2508_21230_b200.dataset import synthetic_rows

SYNTH = ["uniform_700x45", "spec_512x128", "ragged_130x17", "wide_300x64", "c1_slice_1024x128"]


def test_f16_conversion_matches_reference(golden, oracle):
    v16, norms, first = oracle.to_half(golden["tohalf_in"])
    assert first == -1
    assert np.array_equal(v16.view(np.uint16), golden["tohalf_values"])
    assert np.array_equal(norms, golden["tohalf_norms"])


def test_f16_conversion_random_bits(oracle):
    rng = np.random.default_rng(0)
    x = (rng.standard_normal(20000) * np.exp2(rng.integers(-30, 16, 20000))).astype(np.float32)
    x = x[np.abs(x) < 65504]
    L = oracle.lib()
    got = np.array([L.oracle_f32_to_f16(float(v)) for v in x], np.uint16)
    assert np.array_equal(got, x.astype(np.float16).view(np.uint16))


def test_overflow_index(oracle):
    x = np.array([[1.0, 2.0], [3.0, 70000.0]], np.float32)
    _, _, first = oracle.to_half(x)
    assert first == 3   # point 1, dimension 1 (dataset.py:177-183)


def test_frozen_norm_known_answer(oracle):
    # test_dataset.py:172-176: 16 x FP16(0.1) -> 0.15992188
    _, norms, _ = oracle.to_half(np.full((1, 16), 0.1, np.float32))
    assert norms[0] == np.float32(0.15992188)


@pytest.mark.parametrize("name", SYNTH)
def test_to_half_matches_reference(golden, oracle, name):
    v16, norms, _ = oracle.to_half(golden[f"{name}_x"])
    assert np.array_equal(v16.view(np.uint16), golden[f"{name}_values"])
    assert np.array_equal(norms, golden[f"{name}_norms"])


@pytest.mark.parametrize("name", SYNTH)
def test_join_matches_reference_bit_exact(golden, golden_meta, oracle, name):
    meta = golden_meta["cases"][name]
    v16 = golden[f"{name}_values"].view(np.float16)
    i, j, d = oracle.join(v16, golden[f"{name}_norms"], meta["n"], meta["epsilon"], threads=4)
    assert np.array_equal(i, golden[f"{name}_i"])
    assert np.array_equal(j, golden[f"{name}_j"])
    assert np.array_equal(d.view(np.uint32), golden[f"{name}_d"].view(np.uint32))
    assert hashlib.sha256(oracle.pairs_payload(i, j, d)).hexdigest() == meta["result_sha256"]


@pytest.mark.parametrize("name", ["uniform_700x45", "ragged_130x17"])
def test_numpy_restatement_matches_c(golden, golden_meta, oracle, name):
    meta = golden_meta["cases"][name]
    v16 = golden[f"{name}_values"].view(np.float16)
    i, j, d = oracle.join_numpy(v16, golden[f"{name}_norms"], meta["n"], meta["epsilon"])
    assert np.array_equal(i, golden[f"{name}_i"]) and np.array_equal(j, golden[f"{name}_j"])
    assert np.array_equal(d.view(np.uint32), golden[f"{name}_d"].view(np.uint32))


def test_add_rz_restatement():
    from oracle.oracle import add_rz

    a, b = np.float32(1.0), np.float32(3 * 2.0 ** -25)
    assert add_rz(a, b) == np.float32(1.0)             # test_mma.py:27-32
    assert add_rz(-a, -b) == np.float32(-1.0)
    big = np.float32(3.4e38)
    assert add_rz(big, big) == np.finfo(np.float32).max  # saturates (test_mma.py:46-50)


@pytest.mark.parametrize("case,eps", [("integer", 6.0), ("tri", 5.0), ("same", 0.5), ("dup", 0.0)])
def test_small_fixtures(golden, oracle, case, eps):
    x = {"integer": golden.get("integer_x"),
         "tri": np.array([[0.0, 0.0], [3.0, 4.0]], np.float32),
         "same": np.ones((3, 4), np.float32) * 0.7,
         "dup": golden.get("dup_x")}[case]
    v16, norms, _ = oracle.to_half(x)
    i, j, d = oracle.join(v16, norms, x.shape[0], eps, threads=2)
    assert np.array_equal(i, golden[f"{case}_i"]) and np.array_equal(j, golden[f"{case}_j"])
    assert np.array_equal(d.view(np.uint32), golden[f"{case}_d"].view(np.uint32))


def test_tri_and_identical_semantics(golden):
    # SPEC.md:280-282 (3-4-5 inclusive), SPEC.md:410 (3 identical -> S = 2)
    assert list(zip(golden["tri_i"], golden["tri_j"])) == [(1, 1), (1, 2), (2, 1), (2, 2)]
    assert len(golden["same_i"]) == 9


def test_compute_block_tile_fixture(golden, oracle):
    x = golden["tile_x"]
    v16, norms, _ = oracle.to_half(x)
    i, j, d = oracle.join(v16, norms, x.shape[0], float(np.float32(3.3)),
                          rows=(256, 384), cols=(128, 256), threads=2)
    assert np.array_equal(i, golden["tile_i"]) and np.array_equal(j, golden["tile_j"])
    assert np.array_equal(d.view(np.uint32), golden["tile_d"].view(np.uint32))


def test_c1_known_answer(golden_meta, oracle):
    """The full 16K x 128 oracle config reproduces the reference's digest."""
    c1 = golden_meta["C1"]
    x = synthetic_rows(c1["n"], c1["d"], c1["seed"], 0, c1["n"])
    v16, norms, _ = oracle.to_half(x)
    i, j, d = oracle.join(v16, norms, c1["n"], c1["epsilon"])
    assert len(i) == c1["pairs"] == 1199444
    assert hashlib.sha256(oracle.pairs_payload(i, j, d)).hexdigest() == c1["result_sha256"]


def _tile_reference(oracle, n, d, seed, eps, rb, cb):
    """Oracle pairs of tile (rb, cb) from the two 128-row panels only."""
    a = synthetic_rows(n, d, seed, rb * 128, min(rb * 128 + 128, n))
    b = synthetic_rows(n, d, seed, cb * 128, min(cb * 128 + 128, n))
    va, na, _ = oracle.to_half(a)
    vb, nb, _ = oracle.to_half(b)
    X = np.concatenate([va, vb])
    S = np.concatenate([na, nb])
    ii, jj = np.meshgrid(np.arange(128), np.arange(128), indexing="ij")
    ii, jj = ii.ravel(), jj.ravel()
    ok = (rb * 128 + ii < n) & (cb * 128 + jj < n)
    ii, jj = ii[ok], jj[ok]
    d2 = oracle.pair_d2(X, S, (ii + 1).astype(np.uint32), (128 + jj + 1).astype(np.uint32))
    keep = d2 <= oracle.eps_sq_of(eps)
    return (ii[keep] + rb * 128 + 1).astype(np.uint32), (jj[keep] + cb * 128 + 1).astype(np.uint32), \
        d2[keep], na, nb


def test_sampled_tiles_match_reference(golden, golden_meta, oracle):
    """C2-C5 shapes: reference compute_block_tile on sampled tiles."""
    for name, rec in golden_meta["sampled_tiles"].items():
        for t in rec["tiles"]:
            rb, cb = t["row_block"], t["col_block"]
            i, j, d, na, nb = _tile_reference(oracle, rec["n"], rec["d"], rec["seed"],
                                              rec["epsilon"], rb, cb)
            key = f"{name}_{rb}_{cb}"
            assert np.array_equal(na, golden[key + "_rownorms"][:len(na)]), key
            assert np.array_equal(nb, golden[key + "_colnorms"][:len(nb)]), key
            assert np.array_equal(i, golden[key + "_i"]), key
            assert np.array_equal(j, golden[key + "_j"]), key
            assert np.array_equal(d.view(np.uint32), golden[key + "_d"].view(np.uint32)), key
