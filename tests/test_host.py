"""CPU tests: host-side API mirror, validation, the C-ABI library surface.
No GPU compute is called here (the product path has no CPU fallback)."""

import ctypes
import os
import re
import struct

import numpy as np
import pytest

import paper_2508_21230_b200 as F
from paper_2508_21230_b200 import _lib, engine
from paper_2508_21230_b200.tiling import _check_engine_inputs

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


# ── C ABI surface ────────────────────────────────────────────────────────


def _header_symbols():
    src = open(os.path.join(ROOT, "include", "fasted.h")).read()
    return sorted(set(re.findall(r"\b(fasted_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_every_header_symbol():
    L = _lib.load()
    syms = _header_symbols()
    assert len(syms) >= 10
    for s in syms:
        assert hasattr(L, s), s
    assert set(syms) == set(_lib.EXPORTS)


def test_library_host_calls_without_gpu():
    L = _lib.load()
    assert L.fasted_abi_version() == 2
    assert L.fasted_strerror(3) == b"value out of FP16 range"
    assert L.fasted_sort_workspace_bytes(1000, 1000) > 0
    # argument validation happens before any device work
    assert L.fasted_join(None, None, 1, 128, 16, 0, 128, 0, 128, 1.0, 0, None, 0,
                         None, None) == _lib.ERR_ARGUMENT
    assert L.fasted_quantize(None, 1, 1, None, 1, 8, None, None, None) == _lib.ERR_ARGUMENT


def test_product_library_is_configuration_free():
    """libfasted.so reads no FASTED_* environment and has no diagnostic flags
    (the only getenv calls are the static CUDA runtime's own); any flag bit
    outside the public set
    is an ArgumentError before any device work.  libfasted_exp.so (the
    experiment build) exports the same ABI."""
    blob = open(_lib.LIB_PATH, "rb").read()
    assert b"FASTED_" not in blob
    L = _lib.load()
    for bad in (64, 256, 512, 1024, 1 << 16, 1 << 18):
        assert L.fasted_join(None, None, 1, 128, 16, 0, 128, 0, 128, 1.0, bad, None, 0,
                             None, None) == _lib.ERR_ARGUMENT
        assert b"unknown flag" in L.fasted_last_error()
    X = _lib.load_experimental()
    for s in _lib.EXPORTS:
        assert hasattr(X, s), s
    assert b"FASTED_CTA_GROUP" in open(_lib.EXP_LIB_PATH, "rb").read()


def test_library_is_sm100a_only():
    out = os.popen(f"cuobjdump -lelf {_lib.LIB_PATH} 2>/dev/null").read()
    if not out:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out.replace("sm_100a", ""))


def test_kernels_use_tcgen05_and_tma():
    sass = os.popen(f"cuobjdump -sass {_lib.LIB_PATH} 2>/dev/null").read()
    if not sass:
        pytest.skip("cuobjdump unavailable")
    for mnemonic in ("UTCHMMA", "UTMALDG", "LDTM", "FFMA.RZ"):
        assert mnemonic in sass, mnemonic


def test_product_path_fails_loudly_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    hd = F.HalfDataset(3, 4, np.zeros((128, 16), np.float16), np.zeros(128, np.float32))
    with pytest.raises(F.DeviceError):
        F.self_join(hd, 1.0)
    with pytest.raises(F.DeviceError):
        F.to_half(F.Dataset(np.ones((2, 2), np.float32)))


def test_product_package_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2508_21230_b200")
    for fn in os.listdir(pkg):
        if fn.endswith(".py"):
            src = open(os.path.join(pkg, fn)).read()
            assert not re.search(r"^\s*(from|import)\s+oracle", src, re.M), fn


# ── API mirror ───────────────────────────────────────────────────────────


def test_tileconfig_validation_matches_reference():
    F.TileConfig().validate()
    for kw in [dict(warp_kslice=8), dict(warp_side=24), dict(block_side=96),
               dict(block_kslice=24), dict(dispatch_square=0), dict(prefetch_depth=3),
               dict(workers=0)]:
        with pytest.raises(F.ConfigError):
            F.TileConfig(**kw).validate()


def test_engine_input_checks():
    hd = F.HalfDataset(5, 5, np.zeros((64, 16), np.float16), np.zeros(64, np.float32))
    with pytest.raises(F.ConfigError):
        _check_engine_inputs(hd, F.TileConfig())
    hd = F.HalfDataset(5, 5, np.zeros((128, 8), np.float16), np.zeros(128, np.float32))
    with pytest.raises(F.ConfigError):
        _check_engine_inputs(hd, F.TileConfig())


def test_rasterize_examples():   # SPEC.md rasterize_tiles examples
    assert [(c.row_block, c.col_block) for c in F.rasterize_tiles(2, 2, 8)] == \
        [(0, 0), (0, 1), (1, 0), (1, 1)]
    order = F.rasterize_tiles(16, 16, 8)
    assert {(c.row_block, c.col_block) for c in order[:64]} == {(r, c) for r in range(8) for c in range(8)}
    o9 = F.rasterize_tiles(9, 9, 8)
    assert len(o9) == 81 and len(set(o9)) == 81


def test_make_result_set_sorts():
    rs = F.make_result_set([2, 1, 1], [1, 3, 2], np.array([0.5, 0.25, 0.125], np.float32), 3, 1.0)
    assert rs.as_tuples() == [(1, 2, 0.125), (1, 3, 0.25), (2, 1, 0.5)]
    assert rs.i.dtype == np.uint32


def test_selectivity_and_flops():
    rs = F.make_result_set([1, 1, 2, 2, 3, 3, 1, 2, 3], [1, 2, 1, 2, 3, 1, 3, 3, 2],
                           np.zeros(9, np.float32), 3, 1.0)
    assert F.selectivity(rs) == 2.0
    assert F.derived_flops(128, 16, 1.0) == 2 * 128 * 128 * 16 / 1e12
    assert F.distance_tflops(1000, 10, 2.0) == 2 * 1000 * 1000 * 10 / 2.0 / 1e12
    with pytest.raises(F.ArgumentError):
        F.derived_flops(1, 1, 0.0)


def test_overlap_examples():   # SPEC.md overlap_accuracy examples
    a = F.make_result_set([1], [1], np.zeros(1, np.float32), 1, 1.0)
    b = F.make_result_set([1, 1], [1, 2], np.zeros(2, np.float32), 1, 1.0)
    assert F.overlap_accuracy(a, a) == 1.0
    assert F.overlap_accuracy(a, b) == 0.5


def test_distance_error_stats_example():
    t = F.make_result_set([1, 2], [2, 1], np.array([1.1 ** 2, 0.9 ** 2], np.float32), 2, 2.0)
    r = F.make_result_set([1, 2], [2, 1], np.array([1.0, 1.0]), 2, 2.0)
    st = F.distance_error_stats(t, r)
    assert abs(st.err_mean) < 1e-6 and abs(st.err_std - 0.1) < 1e-6


def test_band_compare_classification():
    es = 100.0
    ref = (np.array([1, 1, 2], np.uint32), np.array([1, 2, 2], np.uint32),
           np.array([0.0, 99.95, 10.0], np.float32))
    test = (np.array([1, 2, 2], np.uint32), np.array([1, 1, 2], np.uint32),
            np.array([0.0, 99.99, 10.0], np.float32))
    rep = F.band_compare(*test, *ref, es, lambda i, j: np.array([100.05]))
    assert rep.missing_in_band == 1 and rep.extra_in_band == 1 and rep.ok
    rep = F.band_compare(*test, *ref, es, lambda i, j: np.array([150.0]))
    assert rep.extra_out_of_band == 1 and not rep.ok


def test_calibrate_epsilon_matches_reference_procedure():
    ds = F.generate_synthetic(3, 4, seed=0)
    same = np.repeat(ds.values[:1], 3, axis=0)
    cal = F.calibrate_epsilon(same, 2.0)
    assert cal.iterations == 0 and cal.estimated_selectivity == 2.0
    with pytest.raises(F.CalibrationError):
        F.calibrate_epsilon(F.generate_synthetic(10, 4, seed=1), 20.0)


# ── data ─────────────────────────────────────────────────────────────────


def test_generate_synthetic_matches_numpy_stream():
    ds = F.generate_synthetic(7, 5, seed=12345, lo=-1.0, hi=3.0)
    u = np.random.default_rng(12345).random((7, 5), dtype=np.float32)
    assert np.array_equal(ds.values, u * np.float32(4.0) + np.float32(-1.0))


@pytest.mark.parametrize("n,d,r0,r1", [(50, 7, 3, 20), (50, 8, 0, 50), (50, 9, 11, 12), (9, 3, 9, 9)])
def test_synthetic_rows_equals_full(n, d, r0, r1):
    full = F.generate_synthetic(n, d, seed=99).values
    assert np.array_equal(F.synthetic_rows(n, d, 99, r0, r1), full[r0:r1])


def _write_fvecs(path, rows):
    with open(path, "wb") as f:
        for row in rows:
            f.write(struct.pack("<i", len(row)))
            f.write(struct.pack(f"<{len(row)}f", *row))


def test_load_fvecs_roundtrip_and_errors(tmp_path):   # test_dataset.py:34-82
    p = tmp_path / "a.fvecs"
    _write_fvecs(p, [(1.0, 2.0), (3.0, 4.0)])
    assert np.array_equal(F.load_fvecs(p).values, np.array([[1, 2], [3, 4]], np.float32))
    e = tmp_path / "e.fvecs"
    e.write_bytes(b"")
    with pytest.raises(F.FormatError, match="empty"):
        F.load_fvecs(e)
    b = tmp_path / "b.fvecs"
    with open(b, "wb") as f:
        f.write(struct.pack("<i2f", 2, 1.0, 2.0))
        f.write(struct.pack("<i3f", 3, 1.0, 2.0, 3.0))
        f.write(b"\x00" * 4)
    with pytest.raises(F.FormatError, match="inconsistent dimension 3.*offset 12"):
        F.load_fvecs(b)
    t = tmp_path / "t.fvecs"
    with open(t, "wb") as f:
        f.write(struct.pack("<i2f", 2, 1.0, 2.0))
        f.write(struct.pack("<if", 2, 1.0))
    with pytest.raises(F.FormatError, match="truncated record at byte offset 12"):
        F.load_fvecs(t)
    z = tmp_path / "z.fvecs"
    z.write_bytes(struct.pack("<i", 0))
    with pytest.raises(F.FormatError, match="must be >= 1"):
        F.load_fvecs(z)


def test_dataset_invariants():
    for bad in (np.zeros((0, 3), np.float32), np.zeros((3, 0), np.float32)):
        with pytest.raises(F.ArgumentError):
            F.Dataset(bad)
    x = np.ones((2, 2), np.float32)
    x[1, 1] = np.nan
    with pytest.raises(F.ArgumentError):
        F.Dataset(x)


def test_partition_rows():
    assert engine.partition_rows(1024, 3) == [(0, 256), (256, 640), (640, 1024)]
    with pytest.raises(F.ArgumentError):
        engine.partition_rows(1024, 0)


def test_error_hierarchy():
    assert issubclass(F.RangeError, ValueError) and issubclass(F.RangeError, F.MPJoinError)
    assert issubclass(F.AccumulatorOverflow, ArithmeticError)
    assert issubclass(F.DeviceError, RuntimeError)


def test_device_calibration_validates_before_device_use():
    import paper_2508_21230_b200 as F

    hd = F.HalfDataset(4, 16, np.zeros((128, 16), np.float16), np.zeros(128, np.float32))
    with pytest.raises(F.ArgumentError):
        F.calibrate_epsilon_device(hd, 0.0)
    with pytest.raises(F.ArgumentError):
        F.calibrate_epsilon_device(hd, 1.0, sample_blocks=0)
    with pytest.raises(F.CalibrationError):
        F.calibrate_epsilon_device(hd, 10.0)


def test_python_flag_constants_match_header():
    """_lib's flag and status constants are the values include/fasted.h defines."""
    src = open(os.path.join(ROOT, "include", "fasted.h")).read()
    vals = {k: int(v) for k, v in re.findall(r"\b(FASTED_[A-Z_0-9]+)\s*=\s*(\d+)", src)}
    assert vals["FASTED_JOIN_TC"] == _lib.JOIN_TC
    assert vals["FASTED_JOIN_EXACT"] == _lib.JOIN_EXACT
    assert vals["FASTED_JOIN_COUNT"] == _lib.JOIN_COUNT
    assert vals["FASTED_JOIN_SYMMETRIC"] == _lib.JOIN_SYMMETRIC
    assert vals["FASTED_JOIN_LOW_OUTPUT"] == _lib.JOIN_LOW_OUTPUT
    assert vals["FASTED_JOIN_APPEND"] == _lib.JOIN_APPEND
    assert vals["FASTED_JOIN_SPARSE"] == _lib.JOIN_SPARSE
    assert vals["FASTED_ERR_ARGUMENT"] == _lib.ERR_ARGUMENT
    rec = re.search(r"#define FASTED_RECORD_CHUNK (\d+)", src)
    assert int(rec.group(1)) == engine.RECORD_CHUNK


def test_plan_row_chunks():
    """Contiguous 128-aligned chunks covering the range; count from the
    record budget, at least min_chunks, at most one per row block."""
    ch = engine.plan_row_chunks((0, 1000064), 49e6, 20e6, 1)
    assert len(ch) == 3 and ch[0][0] == 0 and ch[-1][1] == 1000064
    assert all(a[1] == b[0] for a, b in zip(ch, ch[1:]))
    assert all(c[0] % 128 == 0 and c[1] % 128 == 0 for c in ch)
    assert len(engine.plan_row_chunks((0, 1000064), 1e3, 1e9, 4)) == 4
    assert engine.plan_row_chunks((256, 512), 1e9, 1, 1) == [(256, 384), (384, 512)]
    assert engine.plan_row_chunks((128, 128), 10, 1, 4) == [(128, 128)]


def test_taper_chunks():
    """k >= 2 equal chunks -> k + 1 contiguous 128-aligned chunks, first and
    last half-size, none larger than the equal split."""
    eq = engine.plan_row_chunks((0, 1000064), 49e6, 1e9, 2)
    ch = engine.taper_chunks(eq)
    assert len(ch) == 3 and ch[0][0] == 0 and ch[-1][1] == 1000064
    assert all(a[1] == b[0] for a, b in zip(ch, ch[1:]))
    assert all(c[0] % 128 == 0 and c[1] % 128 == 0 for c in ch)
    size = [b - a for a, b in ch]
    assert max(size) <= max(b - a for a, b in eq) and size[0] * 2 <= size[1] + 128
    assert engine.taper_chunks([(0, 1024)]) == [(0, 1024)]
    assert engine.taper_chunks([(0, 128), (128, 256)]) == [(0, 128), (128, 256)]
    four = engine.taper_chunks(engine.plan_row_chunks((256, 256 + 128 * 1000), 1e9, 3e8, 1))
    assert len(four) == 5 and four[0][0] == 256 and four[-1][1] == 256 + 128 * 1000


def test_kernel_selection_rule_is_host_side(monkeypatch):
    """fasted_join_kernel_name applies the launch's selection rule without a
    GPU: resident pair for d_pad <= 512, the CTA pair for large low-output
    joins, multicast clusters otherwise, the exact kernel for mode exact.
    The product library reads no environment: the experiment build's
    overrides, set here, change nothing."""
    L = _lib.load()
    for k, v in (("FASTED_RES_HIT", "0"), ("FASTED_MC_HIT", "0"), ("FASTED_STREAM_HIT", "0"),
                 ("FASTED_STREAM_EPI", "8"), ("FASTED_RES_MAXD", "64"), ("FASTED_RES_EPI", "8"),
                 ("FASTED_MC_EPI", "8"), ("FASTED_CTA_GROUP", "1"), ("FASTED_MC", "0"),
                 ("FASTED_RESIDENT", "0"), ("FASTED_TS", "1")):
        monkeypatch.setenv(k, v)

    def name(d, r, c, f):
        return L.fasted_join_kernel_name(d, r, c, f).decode()

    big = 1 << 19
    assert name(128, big, big, 0) == "fasted::tc::join_tc_res_kernel<2>"
    assert name(960, big, big, _lib.JOIN_LOW_OUTPUT) == "fasted::tc::join_tc_kernel<2>"
    assert name(960, big, big, 0) == "fasted::tc::join_tc_mc_kernel"
    assert name(960, 60032, 60032, _lib.JOIN_LOW_OUTPUT) == "fasted::tc::join_tc_mc_kernel"
    assert name(512, 60032, 60032, _lib.JOIN_LOW_OUTPUT) == "fasted::tc::join_tc_res_kernel<2>"
    assert name(528, big, big, 0) == "fasted::tc::join_tc_mc_kernel"
    assert name(960, big, big, _lib.JOIN_EXACT) == "fasted::join_exact_kernel"
    # FASTED_JOIN_SPARSE: hit warps in the resident and multicast forms
    sp = _lib.JOIN_SPARSE
    assert name(128, big, big, sp) == "fasted::tc::join_tc_res_kernel<2> + 2 hit warps"
    assert name(960, big, big, sp) == "fasted::tc::join_tc_mc_kernel + 2 hit warps"
    assert name(960, big, big, sp | _lib.JOIN_LOW_OUTPUT) == \
        "fasted::tc::join_tc_kernel<2> + 2 hit warps"


def test_form_hints_thresholds():
    """Kernel-form hints from the expected output: LOW_OUTPUT at <= 128 (x1.25)
    pairs per row, SPARSE at <= 1 pair per 8192 examined."""
    from paper_2508_21230_b200 import engine

    r = (0, 1_000_064)
    assert engine.form_hints(74_552_502, r, r) == _lib.JOIN_LOW_OUTPUT | _lib.JOIN_SPARSE   # C3
    assert engine.form_hints(49_048_308, r, r) == _lib.JOIN_LOW_OUTPUT | _lib.JOIN_SPARSE   # C4
    c2 = (0, 60_032)
    assert engine.form_hints(3_623_702, c2, c2) == _lib.JOIN_LOW_OUTPUT                    # C2
    shard, cols = (0, 625_024), (0, 5_000_064)
    assert engine.form_hints(2_516_311_890, shard, cols) == 0                              # C5 S4096
    assert engine.form_hints(160_000_000, shard, cols) == _lib.JOIN_SPARSE                  # C5 S256


def test_overlap_vectorised_equals_reference_loop():
    """analysis.overlap_accuracy (vectorised) == the reference's per-point set
    loop (analysis.py:127-147) bit for bit, incl. empty-on-one/both-sides
    points and a point sample."""
    rng = np.random.default_rng(11)
    n = 300
    for trial in range(4):
        def rand_rs(m):
            i = rng.integers(1, n - 20, m)       # points n-19..n have no pairs anywhere
            j = rng.integers(1, n + 1, m)
            key = np.unique((i.astype(np.uint64) << np.uint64(32)) | j.astype(np.uint64))
            return F.make_result_set((key >> np.uint64(32)).astype(np.uint32),
                                     (key & np.uint64(0xFFFFFFFF)).astype(np.uint32),
                                     np.zeros(len(key), np.float32), n, 1.0)
        a, b = rand_rs(2000 + 300 * trial), rand_rs(1800)
        assert F.overlap_accuracy(a, b) == F.analysis.overlap_accuracy_sets(a, b)
        pts = rng.choice(np.arange(1, n + 1), 50, replace=False)
        assert F.overlap_accuracy(a, b, points=pts) == \
            F.analysis.overlap_accuracy_sets(a, b, points=pts)
    empty = F.make_result_set([], [], np.zeros(0, np.float32), n, 1.0)
    assert F.overlap_accuracy(empty, empty) == 1.0
