"""GPU parity tests: the CUDA path through the C ABI against the reference's
golden vectors and the CPU oracle.  Run on a B200 with ``-m gpu``.

Bars (north star): quantise and the exact kernel are bit-exact; the tcgen05
kernel matches the reference pair set exactly for every pair whose reference
dist_sq lies outside the relative band |d2 - eps^2| <= 1e-3 * eps^2.
"""

import hashlib
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

import paper_2508_21230_b200 as F  # noqa: E402
from paper_2508_21230_b200 import _lib, engine  # noqa: E402

SYNTH = ["uniform_700x45", "spec_512x128", "ragged_130x17", "wide_300x64", "c1_slice_1024x128"]
BAND = 1e-3


@pytest.fixture(scope="module", autouse=True)
def device():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device (no CPU fallback exists)")
    _lib.require_device(0)
    return 0


def _band_ok(oracle, hd, rs, ref_i, ref_j, ref_d, eps, band=BAND):
    es = float(oracle.eps_sq_of(eps))
    rep = F.band_compare(rs.i, rs.j, rs.dist_sq, ref_i, ref_j, ref_d, es,
                         lambda i, j: oracle.pair_d2(hd.values, hd.norms, i, j), band=band)
    return rep


def test_loaded_library_is_in_tree():
    F.self_join(F.to_half(F.Dataset(np.eye(3, dtype=np.float32))), 0.5)
    maps = open("/proc/self/maps").read()
    assert os.path.realpath(_lib.LIB_PATH) in maps


@pytest.mark.parametrize("name", SYNTH)
def test_to_half_bit_exact(golden, name):
    hd = F.to_half(F.Dataset(golden[f"{name}_x"]))
    assert np.array_equal(hd.values.view(np.uint16), golden[f"{name}_values"])
    assert np.array_equal(hd.norms, golden[f"{name}_norms"])
    assert np.array_equal(F.compute_squared_norms(hd), hd.norms)


def test_to_half_known_answers(golden):
    hd = F.to_half(F.Dataset(golden["tohalf_in"]))
    assert np.array_equal(hd.values.view(np.uint16), golden["tohalf_values"])
    assert np.array_equal(hd.norms, golden["tohalf_norms"])
    hd = F.to_half(F.Dataset(np.full((1, 16), 0.1, np.float32)))
    assert hd.norms[0] == np.float32(0.15992188)


def test_range_error_message(golden_meta):
    with pytest.raises(F.RangeError) as e:
        F.to_half(F.Dataset(np.array([[1.0, 2.0], [3.0, 70000.0]], np.float32)))
    assert str(e.value) == golden_meta["range_error_message"]
    with pytest.raises(F.RangeError) as e:
        F.to_half(F.Dataset(np.array([[65520.0]], np.float32)))
    assert str(e.value) == golden_meta["range_error_message_65520"]


def test_to_half_large_matches_oracle(oracle):
    x = F.synthetic_rows(1000000, 960, 12345, 0, 3000)
    x[7, 5] = -60000.0
    x[11, 3] = 2.0 ** -20
    hd = F.to_half(F.Dataset(x))
    v16, norms, _ = oracle.to_half(x)
    assert np.array_equal(hd.values.view(np.uint16), v16.view(np.uint16))
    assert np.array_equal(hd.norms, norms)


@pytest.mark.parametrize("n,d", [(1000, 64), (777, 100), (130, 8), (300, 1024), (5, 4),
                                 (2000, 384), (129, 4100)])
def test_quantize_tma_path_matches_oracle(oracle, n, d):
    """The TMA-streamed quantise kernel (d % 4 == 0): FP16 bits and RZ norms
    equal the oracle's for ragged n, d_pad not a multiple of the 32-column
    box, wide rows and a tiny matrix; the first overflow is reported by flat
    index (RangeError names the lowest point/dimension)."""
    rng = np.random.default_rng(n * 7 + d)
    x = (rng.standard_normal((n, d)) * 50).astype(np.float32)
    x[0, 0] = 1e-6
    x[min(3, n - 1), d // 2] = -65504.0
    hd = F.to_half(F.Dataset(x))
    v16, norms, _ = oracle.to_half(x)
    assert np.array_equal(hd.values.view(np.uint16), v16.view(np.uint16))
    assert np.array_equal(hd.norms, norms)
    y = x.copy()
    y[n - 1, d - 1] = 70000.0
    if n > 2:
        y[n // 2, min(3, d - 1)] = -1e6
    with pytest.raises(F.RangeError) as e:
        F.to_half(F.Dataset(y))
    i, k = (n // 2, min(3, d - 1)) if n > 2 else (n - 1, d - 1)
    assert f"of point {i} (dimension {k})" in str(e.value)


# ── exact kernel: bit parity ─────────────────────────────────────────────


@pytest.mark.parametrize("name", SYNTH)
def test_exact_join_bit_exact(golden, golden_meta, oracle, name):
    meta = golden_meta["cases"][name]
    hd = F.to_half(F.Dataset(golden[f"{name}_x"]))
    rs = F.self_join(hd, meta["epsilon"], mode="exact")
    assert np.array_equal(rs.i, golden[f"{name}_i"])
    assert np.array_equal(rs.j, golden[f"{name}_j"])
    assert np.array_equal(rs.dist_sq.view(np.uint32), golden[f"{name}_d"].view(np.uint32))
    assert hashlib.sha256(oracle.pairs_payload(rs.i, rs.j, rs.dist_sq)).hexdigest() == \
        meta["result_sha256"]


def test_exact_c1_reference_digest(golden_meta, oracle):
    c1 = golden_meta["C1"]
    hd = F.to_half(F.generate_synthetic(c1["n"], c1["d"], seed=c1["seed"]))
    rs = F.self_join(hd, c1["epsilon"], mode="exact")
    assert len(rs) == c1["pairs"]
    assert hashlib.sha256(oracle.pairs_payload(rs.i, rs.j, rs.dist_sq)).hexdigest() == \
        c1["result_sha256"]


def test_compute_block_tile_exact(golden):
    hd = F.to_half(F.Dataset(golden["tile_x"]))
    es = np.float32(np.float32(3.3) * np.float32(3.3))
    i, j, d = F.compute_block_tile(hd, F.TileCoord(2, 1), es, F.TileConfig())
    assert np.array_equal(i, golden["tile_i"]) and np.array_equal(j, golden["tile_j"])
    assert np.array_equal(d.view(np.uint32), golden["tile_d"].view(np.uint32))


def _panel_join(n, d, seed, eps, rb, cb, exact):
    """Join of tile (rb, cb) of a big synthetic shape from its two panels."""
    a = F.synthetic_rows(n, d, seed, rb * 128, min(rb * 128 + 128, n))
    b = F.synthetic_rows(n, d, seed, cb * 128, min(cb * 128 + 128, n))
    pa = np.zeros((128, d), np.float32)
    pb = np.zeros((128, d), np.float32)
    pa[:len(a)], pb[:len(b)] = a, b
    hd = F.to_half(F.Dataset(np.concatenate([pa, pb])))
    dd = engine.upload(hd, 0)
    es = float(np.float32(np.float32(eps) * np.float32(eps)))
    res = engine.join_device(dd, es, rows=(0, 128), cols=(128, 256), exact=exact)
    i, j, dist = engine.to_host(res)
    gi = i.astype(np.int64) - 1 + rb * 128
    gj = j.astype(np.int64) - 1 - 128 + cb * 128
    keep = (i <= len(a)) & (j - 128 <= len(b))
    return (gi[keep] + 1).astype(np.uint32), (gj[keep] + 1).astype(np.uint32), dist[keep], hd


def test_sampled_tiles_exact_and_tc(golden, golden_meta, oracle):
    """C2-C5 shapes, reference compute_block_tile outputs."""
    for name, rec in golden_meta["sampled_tiles"].items():
        for t in rec["tiles"]:
            rb, cb = t["row_block"], t["col_block"]
            key = f"{name}_{rb}_{cb}"
            i, j, d, _ = _panel_join(rec["n"], rec["d"], rec["seed"], rec["epsilon"], rb, cb, True)
            assert np.array_equal(i, golden[key + "_i"]), key
            assert np.array_equal(j, golden[key + "_j"]), key
            assert np.array_equal(d.view(np.uint32), golden[key + "_d"].view(np.uint32)), key
            ti, tj, td, hd = _panel_join(rec["n"], rec["d"], rec["seed"], rec["epsilon"], rb, cb,
                                         False)
            es = float(oracle.eps_sq_of(rec["epsilon"]))

            def ref_d2(a, b, hd=hd, rb=rb, cb=cb):
                # reference dist_sq of TC extras, from the two-panel dataset
                # (row block rb = panel rows 1..128, column block cb = 129..256)
                la = np.asarray(a, np.int64) - rb * 128
                lb = np.asarray(b, np.int64) - cb * 128 + 128
                return oracle.pair_d2(hd.values, hd.norms, la.astype(np.uint32),
                                      lb.astype(np.uint32))

            rep = F.band_compare(ti, tj, td, golden[key + "_i"], golden[key + "_j"],
                                 golden[key + "_d"], es, ref_d2)
            assert rep.ok, (key, rep)


# ── tcgen05 kernel: band parity ──────────────────────────────────────────


@pytest.mark.parametrize("name", SYNTH)
def test_tc_join_band_parity(golden, golden_meta, oracle, name):
    meta = golden_meta["cases"][name]
    hd = F.to_half(F.Dataset(golden[f"{name}_x"]))
    rs = F.self_join(hd, meta["epsilon"])
    rep = _band_ok(oracle, hd, rs, golden[f"{name}_i"], golden[f"{name}_j"],
                   golden[f"{name}_d"], meta["epsilon"])
    assert rep.ok, rep
    assert rep.max_rel_dd2_matched < BAND, rep
    # canonical order
    key = rs.i.astype(np.uint64) << np.uint64(32) | rs.j.astype(np.uint64)
    assert np.all(np.diff(key.astype(np.int64)) > 0)


def test_tc_integer_regime_exact(golden):
    """Small-integer coordinates: every product and partial sum is exact, so
    the tensor core must agree bit for bit (SPEC.md:526 criterion 4)."""
    hd = F.to_half(F.Dataset(golden["integer_x"]))
    rs = F.self_join(hd, 6.0)
    assert np.array_equal(rs.i, golden["integer_i"]) and np.array_equal(rs.j, golden["integer_j"])
    assert np.array_equal(rs.dist_sq, golden["integer_d"])


def test_tc_hand_fixtures(golden):
    tri = F.to_half(F.Dataset(np.array([[0.0, 0.0], [3.0, 4.0]], np.float32)))
    rs = F.self_join(tri, 5.0)
    assert rs.as_tuples() == [(1, 1, 0.0), (1, 2, 25.0), (2, 1, 25.0), (2, 2, 0.0)]
    same = F.to_half(F.Dataset(np.ones((3, 4), np.float32) * 0.7))
    assert F.selectivity(F.self_join(same, 0.5)) == 2.0


@pytest.mark.parametrize("mode", ["tc", "exact"])
def test_eps_zero_gives_self_pairs(mode):
    hd = F.to_half(F.generate_synthetic(3000, 96, seed=5))
    rs = F.self_join(hd, 0.0, mode=mode)
    assert len(rs) == 3000
    assert np.array_equal(rs.i, np.arange(1, 3001, dtype=np.uint32))
    assert np.array_equal(rs.i, rs.j) and not rs.dist_sq.any()


def test_duplicates_eps_zero(golden):
    hd = F.to_half(F.Dataset(golden["dup_x"]))
    rs = F.self_join(hd, 0.0, mode="exact")
    assert np.array_equal(rs.i, golden["dup_i"]) and np.array_equal(rs.j, golden["dup_j"])
    tc = F.self_join(hd, 0.0)
    # the augment step uses the tensor core's own a_ii as norms, so an exact
    # duplicate gives D = a - a/2 - a/2 = 0, i.e. distance 0, as in the
    # reference (whose a_ij and s_i are the same RZ chain)
    assert tc.index_pairs() == rs.index_pairs()
    assert not tc.dist_sq.any()


def test_large_eps_duplicates_and_dist_error():
    """eps^2 >> the squared norms (points in a 0.01-wide cube, eps = 10):
    every pair qualifies; the D = (eps^2 - d2)/2 form reports dist_sq with an
    absolute error of a few ulp(eps^2) -- the augment rows carry
    eps^2/2 + sigma_j exactly (TwoSum), what remains is the tensor core's
    own FP32 summation -- so exact duplicates i != j (reference: 0) come out
    at 0 or 1 ulp(eps^2) (measured on B200: 7.6e-6 at eps^2 = 100)."""
    rng = np.random.default_rng(4)
    x = (rng.random((600, 48)) * 0.01).astype(np.float32)
    x[300:350] = x[0:50]                  # 50 exact duplicate pairs (both orders)
    hd = F.to_half(F.Dataset(x))
    ref = F.self_join(hd, 10.0, mode="exact")
    tc = F.self_join(hd, 10.0)
    assert len(ref) == len(tc) == 600 * 600
    assert tc.same_pairs(ref)
    dup = (np.abs(tc.i.astype(np.int64) - tc.j.astype(np.int64)) == 300) & \
        (np.minimum(tc.i, tc.j) <= 50)
    assert dup.sum() == 100
    ulp = np.spacing(np.float32(100.0))
    assert tc.dist_sq[dup].max() <= ulp, tc.dist_sq[dup].max()
    err = np.abs(tc.dist_sq.astype(np.float64) - ref.dist_sq.astype(np.float64))
    assert err.max() <= 4 * ulp, err.max() / ulp


def test_eps_beyond_fp32_square_returns_all_pairs():
    """An epsilon whose FP32 square overflows (the reference's eps_sq = inf)
    selects every pair, as the reference does: eps_sq clamps to FLT_MAX."""
    hd = F.to_half(F.generate_synthetic(300, 16, seed=2))
    for eps in (2e19, 1e39):
        rs = F.self_join(hd, eps)
        assert len(rs) == 300 * 300
        assert len(F.self_join(hd, eps, mode="exact")) == 300 * 300


def test_c1_tc_vs_reference(golden_meta, oracle):
    c1 = golden_meta["C1"]
    hd = F.to_half(F.generate_synthetic(c1["n"], c1["d"], seed=c1["seed"]))
    ref = F.self_join(hd, c1["epsilon"], mode="exact")   # == reference (digest test)
    st = F.EngineStats()
    rs = F.self_join(hd, c1["epsilon"], stats_out=st)
    rep = _band_ok(oracle, hd, rs, ref.i, ref.j, ref.dist_sq, c1["epsilon"])
    print("C1 band report:", rep, "kernel s:", st.kernel_wall_seconds)
    assert rep.ok, rep


def test_row_sharding_matches_single_device(golden_meta):
    c1 = golden_meta["C1"]
    hd = F.to_half(F.generate_synthetic(5000, 128, seed=3))
    one = F.self_join(hd, 3.9)
    three = F.self_join(hd, 3.9, devices=[0, 0, 0])
    assert one.same_pairs(three)
    assert np.array_equal(one.dist_sq.view(np.uint32), three.dist_sq.view(np.uint32))


def test_capacity_rerun_and_count_only():
    hd = F.to_half(F.generate_synthetic(4000, 64, seed=9))
    dd = engine.upload(hd, 0)
    es = float(np.float32(np.float32(2.6) ** 2))
    full = engine.join_device(dd, es)
    small = engine.join_device(dd, es, capacity=17)
    assert small.reruns >= 1 and small.count == full.count
    a, b = engine.to_host(full), engine.to_host(small)
    assert all(np.array_equal(x, y) for x, y in zip(a, b))
    cnt = torch.zeros(2, dtype=torch.int64, device="cuda:0")
    engine.join_raw(dd, es, _lib.JOIN_COUNT, (0, dd.n_dev), (0, dd.n_dev), None, 0, cnt,
                    torch.cuda.current_stream().cuda_stream)
    assert int(cnt[0].item()) == full.count
    # raw (unsorted) records hold exactly the sorted set, unused slots marked i == 0
    raw = engine.join_device(dd, es, sort=False)
    ri, rj, rd = engine.to_host(raw)
    order = np.lexsort((rj, ri))
    assert np.array_equal(ri[order], a[0]) and np.array_equal(rj[order], a[1])
    assert raw.slots % 256 == 0 and raw.slots >= raw.count


def test_exact_kernel_matches_oracle_at_size(oracle):
    """Bit parity of the exact kernel over a ragged multi-tile problem."""
    x = F.synthetic_rows(10000, 77, 5, 0, 3001)
    hd = F.to_half(F.Dataset(x))
    rs = F.self_join(hd, 2.9, mode="exact")
    oi, oj, od = oracle.join(hd.values, hd.norms, 3001, 2.9)
    assert np.array_equal(rs.i, oi) and np.array_equal(rs.j, oj)
    assert np.array_equal(rs.dist_sq.view(np.uint32), od.view(np.uint32))


def test_long_rows_sort_path():
    """eps above the diameter: every row holds all n pairs (> 1024 -> bitmap path)."""
    n = 2500
    hd = F.to_half(F.generate_synthetic(n, 32, seed=1))
    rs = F.self_join(hd, 100.0)
    assert len(rs) == n * n
    assert np.array_equal(rs.i, np.repeat(np.arange(1, n + 1, dtype=np.uint32), n))
    assert np.array_equal(rs.j, np.tile(np.arange(1, n + 1, dtype=np.uint32), n))


def test_invalid_arguments_raise():
    hd = F.to_half(F.generate_synthetic(10, 8, seed=1))
    with pytest.raises(F.ArgumentError):
        F.self_join(hd, -1.0)
    with pytest.raises(F.ConfigError):
        F.self_join(hd, 1.0, F.TileConfig(warp_kslice=8))
    with pytest.raises(F.ArgumentError):
        F.compute_block_tile(hd, F.TileCoord(5, 0), 1.0, F.TileConfig())


def _exact_and_tc_vs_oracle_blocks(oracle, hd, n, eps, ref, rs, blocks=16):
    """On `blocks` random 128-row blocks (plus the first and the last) at the
    full column range: the exact kernel's records equal the C oracle's bit
    for bit, and the tcgen05 records meet the band contract against the
    oracle directly."""
    nblk = -(-n // 128)
    rng = np.random.default_rng(n + hd.d_padded)
    picks = sorted({0, nblk - 1} | set(rng.choice(nblk, blocks, replace=False).tolist()))
    es = float(oracle.eps_sq_of(eps))
    for rb in picks:
        lo, hi = rb * 128, min(rb * 128 + 128, n)
        oi, oj, od = oracle.join(hd.values, hd.norms, n, eps, rows=(lo, hi))
        sel = (ref.i > lo) & (ref.i <= hi)
        assert np.array_equal(oi, ref.i[sel]) and np.array_equal(oj, ref.j[sel]), rb
        assert np.array_equal(od.view(np.uint32), ref.dist_sq[sel].view(np.uint32)), rb
        tsel = (rs.i > lo) & (rs.i <= hi)
        rep = F.band_compare(rs.i[tsel], rs.j[tsel], rs.dist_sq[tsel], oi, oj, od, es,
                             lambda i, j: oracle.pair_d2(hd.values, hd.norms, i, j))
        assert rep.ok, (rb, rep)
    return picks


@pytest.mark.slow
def test_c3_full_size_tc_vs_exact(oracle):
    """1M x 128 (C3): full tcgen05 join against the bit-exact kernel (itself
    pinned to the reference), plus oracle cross-check of sampled row blocks."""
    n, d, eps = 1000000, 128, 3.685431479161428
    hd = F.to_half(F.generate_synthetic(n, d, seed=12345))
    es = float(oracle.eps_sq_of(eps))
    ref = F.self_join(hd, eps, mode="exact")
    rs = F.self_join(hd, eps)
    rep = _band_ok(oracle, hd, rs, ref.i, ref.j, ref.dist_sq, eps)
    print("C3 band report:", rep)
    assert rep.ok, rep
    _exact_and_tc_vs_oracle_blocks(oracle, hd, n, eps, ref, rs)
    assert es > 0


@pytest.mark.parametrize("n_rows,maxc", [(5000, 150), (20000, 100), (3000, 2000),
                                         (1500, 9000), (200, 20000)])
def test_sort_pairs_random_records(n_rows, maxc):
    """fasted_sort_pairs on shuffled records with unused slots (i == 0):
    short rows (<= 256: warp rank path), mid rows (<= 8192: CTA bitonic
    sort) and long rows (> 8192: bitmap path)."""
    rng = np.random.default_rng(n_rows)
    counts = rng.integers(0, maxc, n_rows)
    i = np.repeat(np.arange(1, n_rows + 1), counts).astype(np.int32)
    n_cols = max(n_rows * 2, 3 * maxc)
    j = np.concatenate([rng.choice(n_cols, c, replace=False) + 1 for c in counts]).astype(np.int32)
    d = rng.random(len(i)).astype(np.float32)
    rec = np.zeros((len(i) + 777, 4), np.int32)
    slots = rng.permutation(len(rec))[:len(i)]
    rec[slots, 0], rec[slots, 1], rec[slots, 2] = i, j, d.view(np.int32)
    L = _lib.load()
    trec = torch.from_numpy(rec).cuda()
    oi, oj = torch.empty(len(i), dtype=torch.int32, device="cuda"), torch.empty(len(i), dtype=torch.int32, device="cuda")
    od = torch.empty(len(i), dtype=torch.float32, device="cuda")
    tjd = torch.empty(len(i), dtype=torch.int64, device="cuda")   # 8-byte (j, d) scratch
    wsb = L.fasted_sort_workspace_bytes(n_rows, n_cols)
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    _lib.check(L.fasted_sort_pairs(trec.data_ptr(), len(rec), 0, n_rows, n_cols, oi.data_ptr(),
                                   oj.data_ptr(), od.data_ptr(), tjd.data_ptr(), tjd.numel() * 8,
                                   ws.data_ptr(), wsb, torch.cuda.current_stream().cuda_stream),
               "sort")
    order = np.lexsort((j, i))
    assert np.array_equal(oi.cpu().numpy(), i[order])
    assert np.array_equal(oj.cpu().numpy(), j[order])
    assert np.array_equal(od.cpu().numpy(), d[order])


class _env:
    """Temporarily set libfasted_exp.so's kernel-form overrides (read per launch)."""

    def __init__(self, **env):
        self.env = {k: str(v) for k, v in env.items()}

    def __enter__(self):
        self.old = {k: os.environ.get(k) for k in self.env}
        os.environ.update(self.env)

    def __exit__(self, *a):
        for k, v in self.old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def _tc_variant(hd, eps, rows=None, cols=None, flags=0, **env):
    """One tcgen05 join through libfasted_exp.so with kernel-form overrides
    (the product library reads no environment: test_product_library_* pins
    its records to these)."""
    with _env(**env):
        dd = engine.upload(hd, 0)
        es = float(np.float32(np.float32(eps) ** 2))
        return engine.to_host(engine.join_device(dd, es, rows=rows, cols=cols, flags=flags,
                                                 lib=_lib.load_experimental()))


def _same(a, b):
    return all(np.array_equal(np.asarray(x).view(np.uint32), np.asarray(y).view(np.uint32))
               for x, y in zip(a, b))


@pytest.mark.parametrize("n,d,eps", [(3000, 128, 3.7), (2999, 100, 3.3), (2000, 512, 8.6),
                                     (1500, 384, 7.7), (3000, 520, 8.5), (1100, 960, 12.0)])
def test_product_library_matches_experiment_forms(n, d, eps):
    """libfasted.so (no environment, no diagnostic flags) gives exactly the
    records of libfasted_exp.so's reference forms -- the streaming kernel
    with one CTA (resident-A at d <= 512 is the same MMA chain) -- with and
    without the SPARSE hint (hit warps) and on a ragged shard range; so every
    bit-identity test below, run on the experiment build, pins the product."""
    hd = F.to_half(F.generate_synthetic(n, d, seed=n + 11 * d))
    ref = _tc_variant(hd, eps, FASTED_CTA_GROUP=1, FASTED_RESIDENT=0)
    assert len(ref[0]) > n
    dd = engine.upload(hd, 0)
    es = float(np.float32(np.float32(eps) ** 2))
    n_dev = dd.n_dev
    for hint in (0, _lib.JOIN_SPARSE, _lib.JOIN_LOW_OUTPUT):
        got = engine.to_host(engine.join_device(dd, es, flags=hint))
        assert _same(ref, got), hint
    rows, cols = (128, min(n_dev, 1152)), (256, n_dev)
    ref = _tc_variant(hd, eps, rows, cols, FASTED_CTA_GROUP=1, FASTED_RESIDENT=0)
    got = engine.to_host(engine.join_device(dd, es, rows=rows, cols=cols))
    assert _same(ref, got)


def test_product_cta_pair_form_matches_single_cta_at_scale():
    """The product's streaming CTA-pair form is chosen only for >= 2^36
    examined pairs with the LOW_OUTPUT hint: run it at that size (256K x 576)
    and compare with libfasted_exp.so's single-CTA streaming kernel."""
    n, d = 262144, 576
    hd = F.to_half(F.generate_synthetic(n, d, seed=3))
    cal = F.calibrate_epsilon_device(hd, 4.0, sample_blocks=8)
    L = _lib.load()
    name = L.fasted_join_kernel_name(hd.d_padded, n, n, _lib.JOIN_LOW_OUTPUT).decode()
    assert "join_tc_kernel<2>" in name, name
    dd = engine.upload(hd, 0)
    es = float(np.float32(np.float32(cal.epsilon) ** 2))
    ref = _tc_variant(hd, cal.epsilon, FASTED_CTA_GROUP=1)
    assert len(ref[0]) > n
    for hint in (_lib.JOIN_LOW_OUTPUT, _lib.JOIN_LOW_OUTPUT | _lib.JOIN_SPARSE):
        got = engine.to_host(engine.join_device(dd, es, flags=hint))
        assert _same(ref, got), hint


def test_product_library_has_no_knobs():
    """No environment variable reaches libfasted.so, and the diagnostic flag
    bits are rejected there (they exist only in libfasted_exp.so)."""
    blob = open(_lib.LIB_PATH, "rb").read()
    assert b"FASTED_" not in blob
    hd = F.to_half(F.generate_synthetic(500, 32, seed=1))
    dd = engine.upload(hd, 0)
    cnt = torch.zeros(2, dtype=torch.int64, device="cuda")
    for bad in (256, 512, 1 << 16, 1 << 20):
        with pytest.raises(F.ArgumentError):
            engine.join_raw(dd, 1.0, _lib.JOIN_COUNT | bad, (0, dd.n_dev), (0, dd.n_dev), None,
                            0, cnt, torch.cuda.current_stream().cuda_stream)


@pytest.mark.parametrize("n,d,eps,seg", [(3000, 128, 3.7, 64), (2999, 100, 3.3, 3),
                                         (1100, 16, 1.0, 1), (2048, 256, 5.6, 2),
                                         (777, 200, 5.0, 64), (5000, 64, 2.6, 7),
                                         (2000, 512, 8.6, 5), (1500, 384, 7.7, 3),
                                         (999, 300, 6.8, 2)])
def test_resident_kernel_bit_identical_to_streaming(n, d, eps, seg):
    """The resident-A kernel (d_pad <= 512) issues the streaming kernel's MMA
    sequence per tile, so every record is bit-identical, for both CTA-group
    forms, ragged segments and ragged row/column ranges."""
    hd = F.to_half(F.generate_synthetic(n, d, seed=n + d))
    for cg in (2, 1):
        ref = _tc_variant(hd, eps, FASTED_RESIDENT=0, FASTED_CTA_GROUP=cg)
        assert len(ref[0]) > n
        for epi, hit in ((16, 0), (8, 0), (16, 2)):
            res = _tc_variant(hd, eps, FASTED_RESIDENT=1, FASTED_CTA_GROUP=cg,
                              FASTED_SEG_TILES=seg, FASTED_RES_EPI=epi, FASTED_RES_HIT=hit)
            for x, y in zip(ref, res):
                assert np.array_equal(x.view(np.uint32), y.view(np.uint32)), (cg, epi, hit, n, d)
    # ragged row ranges x column ranges (the multi-GPU shard shape): the
    # diagonal falls at different offsets inside the 256-column tiles
    n_dev = -(-hd.n_padded // 128) * 128
    for rows, cols in (((128, min(n_dev, 1152)), (256, n_dev)),
                       ((min(n_dev, 384), min(n_dev, 1408)), (128, n_dev)),
                       ((0, n_dev), (min(n_dev, 640), n_dev))):
        ref = _tc_variant(hd, eps, rows, cols, FASTED_RESIDENT=0)
        for hit in (0, 2):
            res = _tc_variant(hd, eps, rows, cols, FASTED_RESIDENT=1, FASTED_SEG_TILES=seg,
                              FASTED_RES_HIT=hit)
            for x, y in zip(ref, res):
                assert np.array_equal(x.view(np.uint32), y.view(np.uint32)), (rows, cols, hit)


@pytest.mark.parametrize("n,d,eps", [(3000, 128, 3.7), (2999, 100, 3.3), (4000, 64, 2.9),
                                     (2000, 512, 8.6), (1500, 384, 7.7)])
def test_resident_hit_warps_symmetric_and_count(n, d, eps):
    """Hit warps (FASTED_RES_HIT=2): the symmetric schedule and the
    count-only join give what the epilogue-warp form gives."""
    hd = F.to_half(F.generate_synthetic(n, d, seed=n * 3 + d))
    es = float(np.float32(np.float32(eps) ** 2))
    dd = engine.upload(hd, 0)
    X = _lib.load_experimental()
    out = {}
    for hit in ("0", "2"):
        with _env(FASTED_RES_HIT=hit):
            rs = engine.to_host(engine.join_device(dd, es, flags=_lib.JOIN_SYMMETRIC, lib=X))
            cnt = torch.zeros(2, dtype=torch.int64, device="cuda")
            engine.join_raw(dd, es, _lib.JOIN_TC | _lib.JOIN_COUNT, (0, dd.n_dev),
                            (0, dd.n_dev), None, 0, cnt, torch.cuda.current_stream().cuda_stream,
                            X)
            out[hit] = (rs, int(cnt[0]))
    (ra, ca), (rb, cb) = out["0"], out["2"]
    # (the full count may exceed the symmetric set by a pair whose D_ij and
    # D_ji straddle the boundary in the last bit; compare like with like)
    assert ca == cb > n and len(ra[0]) == len(rb[0]) > n and abs(ca - len(ra[0])) <= 4
    assert _same(ra, rb)
    # the product library's symmetric schedule gives the same records
    prod = F.self_join(hd, eps, symmetric=True)
    assert _same(ra, (prod.i, prod.j, prod.dist_sq))


@pytest.mark.parametrize("n,d,eps", [(3000, 512, 8.6), (2999, 300, 6.8), (1100, 960, 12.0),
                                     (777, 384, 7.7)])
def test_multicast_kernel_bit_identical_to_single_cta(n, d, eps):
    """The B-multicast cluster kernel (d_pad > 256) issues the single-CTA
    kernel's M=128 MMA sequence per tile: identical bits, including odd
    row-tile counts (a masked partner tile) and ragged shard ranges."""
    hd = F.to_half(F.generate_synthetic(n, d, seed=n * 7 + d))
    ref = _tc_variant(hd, eps, FASTED_CTA_GROUP=1, FASTED_RESIDENT=0)
    assert len(ref[0]) > n
    for mepi, hit in ((8, 0), (16, 0), (16, 2)):
        mc = _tc_variant(hd, eps, FASTED_MC=1, FASTED_CTA_GROUP=0, FASTED_MC_EPI=mepi,
                         FASTED_MC_HIT=hit, FASTED_RES_MAXD=256)
        for x, y in zip(ref, mc):
            assert np.array_equal(x.view(np.uint32), y.view(np.uint32)), mepi
    n_dev = -(-hd.n_padded // 128) * 128
    rows, cols = (128, min(n_dev, 1152)), (256, n_dev)
    ref = _tc_variant(hd, eps, rows, cols, FASTED_CTA_GROUP=1, FASTED_RESIDENT=0)
    mc = _tc_variant(hd, eps, rows, cols, FASTED_MC=1, FASTED_CTA_GROUP=0, FASTED_RES_MAXD=256)
    for x, y in zip(ref, mc):
        assert np.array_equal(x.view(np.uint32), y.view(np.uint32))


@pytest.mark.parametrize("budget", [None, 20000, 3000])
def test_stream_join_pipeline_matches_single_shot(budget, monkeypatch):
    """The row-chunked join -> sort -> D2H pipeline (chunks sized from a
    record budget, double-buffered, D2H on a copy stream) gives exactly the
    single-launch result; a too-low estimate exercises the per-chunk rerun
    and the pinned host buffer growth."""
    hd = F.to_half(F.generate_synthetic(6000, 96, seed=11))
    dd = engine.upload(hd, 0)
    es = float(np.float32(np.float32(3.2) ** 2))
    ref = engine.to_host(engine.join_device(dd, es))
    dd.memo.clear()
    if budget == 3000:
        monkeypatch.setattr(engine, "_estimate_capacity", lambda *a, **k: 10)
        monkeypatch.setattr(engine, "hole_slack", lambda dev: 0)
    host = engine.HostPairs(1)
    kms, sms, reruns, nch = engine.stream_join(dd, es, (0, dd.n_dev), False, host,
                                               budget_records=budget)
    got = host.arrays()
    assert len(got[0]) == len(ref[0]) > 6000
    for x, y in zip(ref, got):
        assert np.array_equal(x.view(np.uint32), y.view(np.uint32))
    if budget == 20000:
        assert nch > 1
    if budget == 3000:
        assert reruns >= 1


@pytest.mark.parametrize("exact", [False, True])
def test_append_flag_sweeps_columns_in_segments(exact):
    """FASTED_JOIN_APPEND: one row range swept in column segments, each
    launch appending to the same record buffer and counts, sorts to exactly
    the single-launch result (tcgen05 and exact kernels)."""
    hd = F.to_half(F.generate_synthetic(5000, 200, seed=5))
    dd = engine.upload(hd, 0)
    es = float(np.float32(np.float32(5.4) ** 2))
    rows = (0, dd.n_dev)
    ref = engine.to_host(engine.join_device(dd, es, rows=rows, exact=exact))
    flags = _lib.JOIN_EXACT if exact else _lib.JOIN_TC
    cap = len(ref[0]) + engine.max_holes(0)
    rec = torch.empty((cap, 4), dtype=torch.int32, device="cuda")
    cnt = torch.zeros(2, dtype=torch.int64, device="cuda")
    s = torch.cuda.current_stream()
    bounds = [0, 1280, 1408, 3840, dd.n_dev]
    for k, (c0, c1) in enumerate(zip(bounds[:-1], bounds[1:])):
        engine.join_raw(dd, es, flags | (_lib.JOIN_APPEND if k else 0), rows, (c0, c1), rec,
                        cap, cnt, s.cuda_stream)
    count, used = (int(v) for v in cnt.tolist())
    assert count == len(ref[0])
    oi, oj, od, _ = engine._sort_records(dd, rec, used * engine.RECORD_CHUNK, count, rows, s)
    got = (oi.cpu().numpy().view(np.uint32), oj.cpu().numpy().view(np.uint32), od.cpu().numpy())
    for x, y in zip(ref, got):
        assert np.array_equal(x.view(np.uint32), y.view(np.uint32))


def test_segmented_upload_pipeline_matches_resident(monkeypatch):
    """upload_segmented + stream_join: the first row chunk sweeps its columns
    segment by segment as the copy lands (FASTED_JOIN_APPEND), later chunks
    run on the resident dataset -- exactly the result of a join on a fully
    resident copy."""
    hd = F.to_half(F.generate_synthetic(9000, 256, seed=8), pin_host=True)
    es = float(np.float32(np.float32(6.0) ** 2))
    dd0 = engine.upload(hd, 0)
    ref = engine.to_host(engine.join_device(dd0, es))
    monkeypatch.setattr(engine, "SEGMENT_MIN_BYTES", 0)
    monkeypatch.setattr(engine, "PIPELINE_MIN_RECORDS", 0)     # 4 row chunks
    if hasattr(hd, "device_cache"):
        hd.device_cache.clear()
    for segments in (8, 3):
        hd.count_memo.clear()
        dd = engine.upload_segmented(hd, 0, segments=segments)
        assert dd.ready is not None and len(dd.ready) == segments
        segs = engine.column_segments(dd, (0, dd.n_dev), dd.n_dev // 4 // 128 * 128)
        assert len(segs) == 2 and segs[0][0] == 0 and segs[-1][1] == dd.n_dev
        assert segs[0][1] < dd.n_dev and segs[1][2] == dd.n_dev
        host = engine.HostPairs(1)
        kms, sms, reruns, nch = engine.stream_join(dd, es, (0, dd.n_dev), False, host)
        assert nch > 1 and dd.ready is None
        got = host.arrays()
        for x, y in zip(ref, got):
            assert np.array_equal(x.view(np.uint32), y.view(np.uint32)), segments


def test_device_calibration_hits_target_on_full_data(golden_meta):
    """GPU count-only bisection (16 row blocks x all columns): the full
    join at the calibrated epsilon lands within a few percent of the target
    selectivity -- the reference's 1024-point FP64 sample gave 72.2 for a
    target of 64 on C1."""
    c1 = golden_meta["C1"]
    hd = F.to_half(F.generate_synthetic(c1["n"], c1["d"], seed=c1["seed"]))
    cal = F.calibrate_epsilon_device(hd, 64.0, tol=0.01, sample_blocks=16)
    assert abs(cal.estimated_selectivity - 64.0) <= 0.64
    assert cal.sample_size == 16 * 128
    rs = F.self_join(hd, cal.epsilon)
    s_full = F.selectivity(rs)
    print("device calibration:", cal, "full-data S:", s_full)
    assert abs(s_full - 64.0) / 64.0 < 0.04
    with pytest.raises(F.CalibrationError):
        F.calibrate_epsilon_device(hd, float(c1["n"]))


@pytest.mark.parametrize("n,d,eps", [(3000, 64, 2.6), (2999, 128, 3.9), (1500, 300, 6.8),
                                     (2100, 960, 12.0)])
@pytest.mark.parametrize("env", [None, {"FASTED_CTA_GROUP": "1"}, {"FASTED_CTA_GROUP": "2",
                                                                    "FASTED_RESIDENT": "0"}])
def test_symmetric_join(oracle, n, d, eps, env):
    """FASTED_JOIN_SYMMETRIC (upper tiles + mirrored records) on every kernel
    form (the product library, and libfasted_exp.so's forced streaming
    forms): the pair set is exactly symmetric with equal dist_sq both ways,
    equals the full join outside the 1e-3 band, and passes the band contract
    against the reference oracle."""
    hd = F.to_half(F.generate_synthetic(n, d, seed=n + 3 * d))
    if env is None:
        full = F.self_join(hd, eps)
        sym = F.self_join(hd, eps, symmetric=True)
    else:
        full = F.make_result_set(*_tc_variant(hd, eps, **env), n, eps)
        sym = F.make_result_set(*_tc_variant(hd, eps, flags=_lib.JOIN_SYMMETRIC, **env), n, eps)
    assert len(sym) > n
    # exact symmetry: (i, j, d) present <=> (j, i, d) present
    key = (sym.i.astype(np.uint64) << np.uint64(32)) | sym.j.astype(np.uint64)
    tkey = (sym.j.astype(np.uint64) << np.uint64(32)) | sym.i.astype(np.uint64)
    o1, o2 = np.argsort(key), np.argsort(tkey)
    assert np.array_equal(key[o1], tkey[o2])
    assert np.array_equal(sym.dist_sq[o1].view(np.uint32), sym.dist_sq[o2].view(np.uint32))
    assert np.all(sym.i[sym.i == sym.j] > 0) and np.all(sym.dist_sq[sym.i == sym.j] == 0)
    es = float(oracle.eps_sq_of(eps))
    rep = F.band_compare(sym.i, sym.j, sym.dist_sq, full.i, full.j, full.dist_sq, es,
                         lambda i, j: oracle.pair_d2(hd.values, hd.norms, i, j))
    assert rep.missing_out_of_band == 0 and rep.extra_out_of_band == 0, rep
    oi, oj, od = oracle.join(hd.values, hd.norms, n, eps)
    rep = _band_ok(oracle, hd, sym, oi, oj, od, eps)
    assert rep.ok, rep


def test_symmetric_rejects_shards_and_exact():
    hd = F.to_half(F.generate_synthetic(500, 32, seed=1))
    with pytest.raises(F.ArgumentError):
        F.self_join(hd, 1.0, symmetric=True, devices=[0, 0])
    with pytest.raises(F.ArgumentError):
        F.self_join(hd, 1.0, symmetric=True, mode="exact")
    with pytest.raises(F.ArgumentError):
        F.self_join(hd, 1.0, symmetric=True, shard=(0, 2))


def test_c2_full_size_band_parity_all_schedules(oracle):
    """C2 (60K x 512) in full: the product path (B-multicast kernel), its
    symmetric schedule and a 3-way row sharding all meet the band contract
    against the bit-exact kernel (itself pinned to the reference), and the
    shards concatenate to the single-device result."""
    n, d, eps = 60000, 512, 8.48414709018062
    hd = F.to_half(F.generate_synthetic(n, d, seed=12345))
    ref = F.self_join(hd, eps, mode="exact")
    tc = F.self_join(hd, eps)
    rep = _band_ok(oracle, hd, tc, ref.i, ref.j, ref.dist_sq, eps)
    print("C2 band report:", rep)
    assert rep.ok, rep
    sym = F.self_join(hd, eps, symmetric=True)
    rep = _band_ok(oracle, hd, sym, ref.i, ref.j, ref.dist_sq, eps)
    assert rep.ok, rep
    parts = [F.self_join(hd, eps, shard=(r, 3)) for r in range(3)]
    assert np.array_equal(np.concatenate([p.i for p in parts]), tc.i)
    assert np.array_equal(np.concatenate([p.j for p in parts]), tc.j)
    assert np.array_equal(np.concatenate([p.dist_sq for p in parts]).view(np.uint32),
                          tc.dist_sq.view(np.uint32))


@pytest.mark.slow
def test_c4_full_size_tc_vs_exact(oracle):
    """The headline configuration in full (1M x 960, the bench's eps): the
    tcgen05 pair set against the bit-exact kernel's (= the reference's
    arithmetic) under the band contract; the exact kernel against the C
    oracle on sampled row blocks at the full column range."""
    n, d, eps = 1000000, 960, 11.700486640655093
    hd = F.to_half(F.generate_synthetic(n, d, seed=12345))
    ref = F.self_join(hd, eps, mode="exact")
    rs = F.self_join(hd, eps)
    rep = _band_ok(oracle, hd, rs, ref.i, ref.j, ref.dist_sq, eps)
    print("C4 band report:", rep)
    assert rep.ok, rep
    _exact_and_tc_vs_oracle_blocks(oracle, hd, n, eps, ref, rs)


def test_cta_pair_low_output_form_matches_single_cta():
    """The large-join form at d_pad > 256 (CTA pair, 16K-row raster, picked
    by the FASTED_JOIN_LOW_OUTPUT hint on >= 2^36 examined pairs) gives the
    single-CTA kernel's bits: per element both accumulate the same K-ordered
    MMA chain.  Also checks the selection rule itself."""
    L = _lib.load()
    name = lambda d, r, c, f: L.fasted_join_kernel_name(d, r, c, f).decode()
    big = 1 << 19
    assert "join_tc_kernel<2>" in name(960, big, big, _lib.JOIN_LOW_OUTPUT)
    assert "mc" in name(960, big, big, 0)
    assert "mc" in name(960, 60032, 60032, _lib.JOIN_LOW_OUTPUT)
    assert "res" in name(128, big, big, _lib.JOIN_LOW_OUTPUT)
    assert "res" in name(512, big, big, _lib.JOIN_LOW_OUTPUT)
    hd = F.to_half(F.generate_synthetic(3000, 520, seed=77))    # d_pad 528: streaming forms
    one = _tc_variant(hd, 8.5, FASTED_CTA_GROUP=1)
    assert len(one[0]) > 3000
    for sepi, hit in ((8, 0), (16, 0), (16, 2)):
        pair = _tc_variant(hd, 8.5, FASTED_CTA_GROUP=2, FASTED_STREAM_EPI=sepi,
                           FASTED_STREAM_HIT=hit)
        for x, y in zip(one, pair):
            assert np.array_equal(x.view(np.uint32), y.view(np.uint32)), (sepi, hit)


@pytest.mark.parametrize("symmetric", [False, True])
def test_pacing_layer_counts_complete(symmetric):
    """Both CTA-pair forms pace their producers on a global count of issued
    tile layers.  The layer count must close on every schedule shape, or a
    producer waits forever (the launch traps after 20 s):
      * streaming pair, 69 x 69 tiles of 256 on 74 pairs (148 SMs): every pair
        has 64 tiles and 25 have 65 -- a last block of exactly 64 layers;
      * resident pair, 79 row tiles x 2 column segments = 158 units on 74
        pairs: a partial last unit layer.
    Records equal the unpaced single-CTA streaming form bit for bit
    (symmetric: tiles skipped below the diagonal still count as layers)."""
    flags = _lib.JOIN_SYMMETRIC if symmetric else 0
    hd = F.to_half(F.generate_synthetic(69 * 256, 520, seed=69))
    one = _tc_variant(hd, 8.6, flags=flags, FASTED_CTA_GROUP=1, FASTED_RESIDENT=0)
    pair = _tc_variant(hd, 8.6, flags=flags, FASTED_CTA_GROUP=2, FASTED_STREAM_PACE_W=1)
    assert len(one[0]) > 69 * 256 and _same(one, pair)
    # multicast clusters: 35 super-rows x 69 column tiles = 2415 tiles on 74 clusters
    mc = _tc_variant(hd, 8.6, flags=flags, FASTED_MC=1, FASTED_CTA_GROUP=0, FASTED_MC_PACE_W=1)
    assert _same(one, mc)
    hd = F.to_half(F.generate_synthetic(20000, 128, seed=79))
    one = _tc_variant(hd, 3.7, flags=flags, FASTED_CTA_GROUP=1, FASTED_RESIDENT=0)
    for w in (1, 2):
        res = _tc_variant(hd, 3.7, flags=flags, FASTED_PACE_W=w, FASTED_SEG_TILES=40)
        assert len(one[0]) > 20000 and _same(one, res), w


def test_concurrent_paced_joins_complete():
    """Two joins launched at once on two streams of one device: each grid
    holds one CTA per SM, so the block scheduler can leave each kernel only
    partly resident.  Pacing must not turn that into a deadlock (a producer
    waiting for CTAs that cannot be scheduled until the other kernel ends): a
    pacing wait gives up after 5 ms.  Both launches finish and each equals the
    same join run alone, bit for bit."""
    import torch

    hd = F.to_half(F.generate_synthetic(60000, 128, seed=61))
    dd = engine.upload(hd, 0)
    es = float(np.float32(np.float32(3.7) ** 2))
    rows, cols = (0, dd.n_dev), (0, dd.n_dev)
    alone = engine.join_device(dd, es, rows=rows, sort=False)
    cap = alone.count + engine.hole_slack(0)
    ref = engine.to_host(engine.join_device(dd, es, rows=rows))
    streams = [torch.cuda.Stream() for _ in range(2)]
    recs = [torch.empty((cap, 4), dtype=torch.int32, device="cuda") for _ in range(2)]
    cnts = [torch.zeros(2, dtype=torch.int64, device="cuda") for _ in range(2)]
    torch.cuda.synchronize()
    for _ in range(3):
        for k in range(2):
            engine.join_raw(dd, es, _lib.JOIN_TC, rows, cols, recs[k], cap, cnts[k],
                            streams[k].cuda_stream)
    torch.cuda.synchronize()
    for k in range(2):
        assert int(cnts[k][0].item()) == alone.count
        slots = int(cnts[k][1].item()) * engine.RECORD_CHUNK
        raw = recs[k][:slots].cpu().numpy()
        raw = raw[raw[:, 0] != 0]
        order = np.lexsort((raw[:, 1].view(np.uint32), raw[:, 0].view(np.uint32)))
        got = (raw[order, 0].view(np.uint32), raw[order, 1].view(np.uint32),
               raw[order, 2].view(np.float32))
        assert _same(ref, got)


def test_sort_long_rows_bucket_and_fallback_paths():
    """Rows above 16384 records: spread j -> column buckets + shared-memory
    bitonic per bucket; j clustered in one bucket -> the bitmap fallback.
    Both must give the reference's lexsort order."""
    rng = np.random.default_rng(5)
    n_cols = 4_000_000
    rows = []
    rows.append(rng.choice(n_cols, 30000, replace=False) + 1)          # spread: bucket path
    rows.append(rng.choice(25000, 20000, replace=False) + 1)           # clustered: fallback
    rows.append(rng.choice(n_cols, 3000, replace=False) + 1)           # mid path
    i = np.concatenate([np.full(len(r), k + 1) for k, r in enumerate(rows)]).astype(np.int32)
    j = np.concatenate(rows).astype(np.int32)
    d = rng.random(len(i)).astype(np.float32)
    perm = rng.permutation(len(i))
    rec = np.zeros((len(i), 4), np.int32)
    rec[:, 0], rec[:, 1], rec[:, 2] = i[perm], j[perm], d[perm].view(np.int32)
    L = _lib.load()
    trec = torch.from_numpy(rec).cuda()
    n = len(i)
    oi, oj = (torch.empty(n, dtype=torch.int32, device="cuda") for _ in range(2))
    od = torch.empty(n, dtype=torch.float32, device="cuda")
    tjd = torch.empty(n, dtype=torch.int64, device="cuda")   # 8-byte (j, d) scratch
    wsb = L.fasted_sort_workspace_bytes(len(rows), n_cols)
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    _lib.check(L.fasted_sort_pairs(trec.data_ptr(), n, 0, len(rows), n_cols, oi.data_ptr(),
                                   oj.data_ptr(), od.data_ptr(), tjd.data_ptr(), tjd.numel() * 8,
                                   ws.data_ptr(), wsb, torch.cuda.current_stream().cuda_stream),
               "sort")
    order = np.lexsort((j, i))
    assert np.array_equal(oi.cpu().numpy(), i[order])
    assert np.array_equal(oj.cpu().numpy(), j[order])
    assert np.array_equal(od.cpu().numpy(), d[order])


def _sort_rows_on_device(rows, n_cols, seed=0):
    """fasted_sort_pairs over shuffled records of the given per-row j lists
    (plus unused slots); returns (expected, got) as (i, j, d) arrays."""
    rng = np.random.default_rng(seed)
    i = np.concatenate([np.full(len(r), k + 1) for k, r in enumerate(rows)]).astype(np.int32)
    j = np.concatenate(rows).astype(np.int32)
    d = rng.random(len(i)).astype(np.float32)
    rec = np.zeros((len(i) + 300, 4), np.int32)
    slots = rng.permutation(len(rec))[:len(i)]
    rec[slots, 0], rec[slots, 1], rec[slots, 2] = i, j, d.view(np.int32)
    L = _lib.load()
    trec = torch.from_numpy(rec).cuda()
    n = len(i)
    oi, oj = (torch.empty(n, dtype=torch.int32, device="cuda") for _ in range(2))
    od = torch.empty(n, dtype=torch.float32, device="cuda")
    tjd = torch.empty(n, dtype=torch.int64, device="cuda")   # 8-byte (j, d) scratch
    wsb = L.fasted_sort_workspace_bytes(len(rows), n_cols)
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    _lib.check(L.fasted_sort_pairs(trec.data_ptr(), len(rec), 0, len(rows), n_cols,
                                   oi.data_ptr(), oj.data_ptr(), od.data_ptr(), tjd.data_ptr(),
                                   tjd.numel() * 8, ws.data_ptr(), wsb,
                                   torch.cuda.current_stream().cuda_stream), "sort")
    order = np.lexsort((j, i))
    return (i[order], j[order], d[order]), (oi.cpu().numpy(), oj.cpu().numpy(), od.cpu().numpy())


def test_sort_rank_paths_and_fallbacks():
    """Every per-row ordering path: warp rank (<= 256), bucketed rank sort
    (<= 4096, <= 16384), its bitonic fallback when one bucket is crowded
    (dense j plus a far outlier), column super-buckets for long rows with a
    rank sort or (crowded super-bucket) bitonic inside, and the bitmap
    fallback for an overfull super-bucket."""
    rng = np.random.default_rng(11)
    n_cols = 4_000_000
    spread = lambda m: rng.choice(n_cols, m, replace=False) + 1
    rows = [
        spread(100),                                                   # warp rank
        spread(3000),                                                  # rank sort <= 4096
        spread(10000),                                                 # rank sort <= 16384
        np.concatenate([np.arange(1, 3000), [n_cols]]),                # crowded: bitonic
        np.concatenate([np.arange(1, 12000), [n_cols - 5]]),           # crowded: bitonic (big)
        spread(40000),                                                 # super-buckets + rank
        np.concatenate([np.arange(1, 15001),                           # super-bucket with a
                        rng.choice(np.arange(15001, n_cols), 5000, replace=False) + 1]),
        np.arange(1, 20001) * 3,                                       # overfull: bitmap
        spread(257), spread(4097), spread(16385),                      # tier boundaries
        np.array([n_cols, 1, 2]),
    ]
    want, got = _sort_rows_on_device(rows, n_cols + 1)
    for x, y in zip(want, got):
        assert np.array_equal(x.view(np.uint32), np.asarray(y).view(np.uint32))


@pytest.mark.parametrize("n,d,eps", [(5, 3, 0.7), (130, 2000, 25.5), (257, 4100, 36.8)])
def test_tc_extreme_shapes_band_parity(oracle, n, d, eps):
    """Tiny n (one partial row block) and large d (k loop of 32-65 blocks,
    ragged last block zero-filled by TMA) on every kernel form."""
    hd = F.to_half(F.generate_synthetic(n, d, seed=d))
    oi, oj, od = oracle.join(hd.values, hd.norms, n, eps)
    for env in ({}, {"FASTED_CTA_GROUP": "1"}, {"FASTED_CTA_GROUP": "2"}):
        got = _tc_variant(hd, eps, **env)
        rs = F.make_result_set(got[0], got[1], got[2], n, eps)
        rep = _band_ok(oracle, hd, rs, oi, oj, od, eps)
        assert rep.ok, (env, rep)
        assert len(rs) >= n


@pytest.mark.parametrize("n,d,eps", [(3000, 128, 3.7), (2999, 100, 3.3), (1100, 16, 1.0),
                                     (5000, 64, 2.6), (777, 120, 3.5)])
def test_tmem_a_kernel_bit_identical(n, d, eps):
    """The TMEM-A kernel (A panel in tensor memory, three 128-column
    accumulators) issues the same per-element K-ordered MMA chain as the
    resident kernel: identical bits, also on a ragged shard range and under
    the symmetric schedule."""
    hd = F.to_half(F.generate_synthetic(n, d, seed=n + 5 * d))
    ref = _tc_variant(hd, eps, FASTED_TS=0)
    assert len(ref[0]) > n
    ts = _tc_variant(hd, eps, FASTED_TS=1)
    for x, y in zip(ref, ts):
        assert np.array_equal(x.view(np.uint32), y.view(np.uint32))
    n_dev = -(-hd.n_padded // 128) * 128
    rows, cols = (128, min(n_dev, 1152)), (256, n_dev)
    ref = _tc_variant(hd, eps, rows, cols, FASTED_TS=0)
    ts = _tc_variant(hd, eps, rows, cols, FASTED_TS=1, FASTED_SEG_TILES=3)
    for x, y in zip(ref, ts):
        assert np.array_equal(x.view(np.uint32), y.view(np.uint32))
    sym = F.make_result_set(*_tc_variant(hd, eps, flags=_lib.JOIN_SYMMETRIC, FASTED_TS=1), n, eps)
    full = F.self_join(hd, eps)
    key = lambda r: set(zip(r.i.tolist(), r.j.tolist()))
    assert len(key(sym) ^ key(full)) <= max(2, len(full) // 10000)


@pytest.mark.slow
def test_c5_rows_at_full_column_range(oracle):
    """C5 (5M x 384) at S ~ 1000: two sampled row blocks against all 5M
    columns -- the exact kernel equals the C oracle bit for bit, and the
    product path meets the band contract against it."""
    n, d, eps = 5_000_000, 384, 7.1352369182727085
    hd = F.to_half(F.generate_synthetic(n, d, seed=12345))
    dd = engine.upload(hd, 0)
    es = float(oracle.eps_sq_of(eps))
    for rb in (0, 23456):
        rows = (rb * 128, rb * 128 + 128)
        ex = engine.to_host(engine.join_device(dd, es, rows=rows, exact=True))
        tc = engine.to_host(engine.join_device(dd, es, rows=rows))
        oi, oj, od = oracle.join(hd.values, hd.norms, n, eps, rows=rows)
        assert np.array_equal(oi, ex[0]) and np.array_equal(oj, ex[1])
        assert np.array_equal(od.view(np.uint32), ex[2].view(np.uint32))
        assert len(ex[0]) > 128 * 500
        rep = F.band_compare(tc[0], tc[1], tc[2], ex[0], ex[1], ex[2], es,
                             lambda i, j: oracle.pair_d2(hd.values, hd.norms, i, j))
        print("C5 row block", rb, rep)
        assert rep.ok, rep


def test_engine_stats_fields():
    """EngineStats (tiling.py:125-151) is filled from device measurements:
    the H2D stage time is the copy's CUDA-event time (a host dataset with no
    device copy must pay it: > 0 and at least the bytes at ~60 GB/s cannot be
    faster than ~1/100 of a second here), kernel time below the wall time,
    the FMA count is n_pad^2 d_pad, per-device phase reports present; a
    dataset already resident (to_half's device cache) stages nothing."""
    hd = F.to_half(F.generate_synthetic(40000, 256, seed=5), pin_host=True)
    host = F.HalfDataset(hd.n_logical, hd.d_logical, hd.values, hd.norms)   # no device cache
    st = F.EngineStats()
    rs = F.self_join(host, 5.2, stats_out=st)
    nbytes = hd.values.nbytes + hd.norms.nbytes
    assert st.stage_seconds > 0 and nbytes / st.stage_seconds < 80e9, (st.stage_seconds, nbytes)
    assert 0 < st.kernel_wall_seconds < st.wall_seconds
    n_dev = -(-hd.n_padded // 128) * 128
    assert st.fma_ops == n_dev * n_dev * hd.d_padded and st.tiles > 0
    dev0 = st.per_device[0]
    for k in ("chunks", "reruns", "sort_ms", "d2h_ms"):
        assert k in dev0, dev0.keys()
    assert dev0["d2h_ms"] > 0 and dev0["sort_ms"] >= 0
    st2 = F.EngineStats()
    rs2 = F.self_join(hd, 5.2, stats_out=st2)      # resident: nothing to stage
    assert st2.stage_seconds == 0.0
    assert rs.same_pairs(rs2)
