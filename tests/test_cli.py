"""CLI drop-in (`join` / `calibrate`): pair-file format, manifest, exit codes."""

import json

import numpy as np
import pytest

import paper_2508_21230_b200 as F
from paper_2508_21230_b200 import cli


def test_pairs_roundtrip(tmp_path):
    rs = F.make_result_set([2, 1, 1], [1, 3, 1], np.array([0.5, 0.25, 0.0], np.float32), 3, 1.0)
    p = tmp_path / "x.pairs"
    digest = cli.write_pairs(p, rs)
    raw = p.read_bytes()
    assert int(np.frombuffer(raw[:8], "<u8")[0]) == 3 and len(raw) == 8 + 3 * 12
    back = cli.read_pairs(p, 3, 1.0)
    assert back.as_tuples() == rs.as_tuples()
    import hashlib
    assert hashlib.sha256(raw).hexdigest() == digest
    p.write_bytes(raw[:-1])
    with pytest.raises(F.FormatError):
        cli.read_pairs(p, 3, 1.0)


def test_dataset_digest_matches_reference(golden_meta):
    c1 = golden_meta["C1"]
    ds = F.generate_synthetic(c1["n"], c1["d"], seed=c1["seed"])
    assert cli.dataset_sha256(ds) == c1["dataset_sha256"]


def test_exit_codes_without_gpu():
    assert cli.main(["join", "--synthetic", "10x0", "--epsilon", "1"]) == cli.EXIT_ARGUMENT
    assert cli.main(["join", "--synthetic", "10x4", "--epsilon", "-1"]) == cli.EXIT_ARGUMENT
    assert cli.main(["join", "--synthetic", "10x4", "--epsilon", "1", "--warp-side", "24"]) == \
        cli.EXIT_ARGUMENT
    assert cli.main(["join", "--fvecs", "/nonexistent.fvecs", "--epsilon", "1"]) == cli.EXIT_FORMAT


def test_calibrate_command(capsys):
    assert cli.main(["calibrate", "--synthetic", "400x8", "--target-selectivity", "5",
                     "--json"]) == cli.EXIT_OK
    out = [json.loads(x) for x in capsys.readouterr().out.strip().splitlines()]
    assert {o["metric"] for o in out} == {"epsilon", "estimated_selectivity", "iterations",
                                          "sample_size"}


@pytest.mark.gpu
def test_join_exact_reproduces_reference_digest(tmp_path, golden_meta, capsys):
    c1 = golden_meta["C1"]
    out = tmp_path / "c1.pairs"
    rc = cli.main(["join", "--synthetic", "16384x128", "--seed", "12345", "--epsilon",
                   repr(c1["epsilon"]), "--mode", "exact", "--pairs-out", str(out), "--json"])
    assert rc == 0
    man = json.loads((tmp_path / "c1.pairs.manifest.json").read_text())
    assert man["result_sha256"] == c1["result_sha256"]
    assert man["pairs"] == c1["pairs"] and man["dataset"]["sha256"] == c1["dataset_sha256"]
    rc = cli.main(["join", "--synthetic", "16384x128", "--epsilon", repr(c1["epsilon"]),
                   "--manifest", str(tmp_path / "tc.json")])
    assert rc == 0
    tc = json.loads((tmp_path / "tc.json").read_text())
    assert abs(tc["pairs"] - c1["pairs"]) < 1e-3 * c1["pairs"]


@pytest.mark.gpu
def test_join_symmetric_and_device_calibration(tmp_path, golden_meta):
    """`join --symmetric` writes the same pairs file format with an exactly
    symmetric pair set close to the full join's; `--target-selectivity` with
    `--calibration-method device` lands near the target on the full data."""
    c1 = golden_meta["C1"]
    for extra, name in (([], "full"), (["--symmetric"], "sym")):
        rc = cli.main(["join", "--synthetic", "16384x128", "--epsilon", repr(c1["epsilon"]),
                       "--pairs-out", str(tmp_path / f"{name}.pairs")] + extra)
        assert rc == 0
    full = cli.read_pairs(tmp_path / "full.pairs", 16384, c1["epsilon"])
    sym = cli.read_pairs(tmp_path / "sym.pairs", 16384, c1["epsilon"])
    assert abs(len(sym) - len(full)) < 1e-3 * len(full)
    assert set(zip(sym.i.tolist(), sym.j.tolist())) == set(zip(sym.j.tolist(), sym.i.tolist()))
    rc = cli.main(["join", "--synthetic", "16384x128", "--target-selectivity", "64",
                   "--calibration-method", "device", "--calibration-tol", "0.01",
                   "--manifest", str(tmp_path / "cal.json")])
    assert rc == 0
    man = json.loads((tmp_path / "cal.json").read_text())
    s = (man["pairs"] - 16384) / 16384
    assert abs(s - 64) / 64 < 0.05, s


def test_accuracy_refuses_mismatched_truth(tmp_path, capsys):
    """`accuracy --truth-pairs` with a manifest recorded for another dataset is
    refused before any compute (cli.py:305-314), exit code 2."""
    rs = F.make_result_set([1], [1], np.zeros(1, np.float32), 50, 1.0)
    p = tmp_path / "truth.pairs"
    cli.write_pairs(p, rs)
    (tmp_path / "truth.pairs.manifest.json").write_text(
        json.dumps({"dataset": {"sha256": "0" * 64}, "epsilon": 1.0}))
    rc = cli.main(["accuracy", "--synthetic", "50x4", "--epsilon", "1",
                   "--truth-pairs", str(p)])
    assert rc == cli.EXIT_ARGUMENT
    assert "dataset hash mismatch" in capsys.readouterr().err


def test_bench_argument_errors():
    assert cli.main(["bench", "--n", "100", "--dims", "0"]) == cli.EXIT_ARGUMENT
    assert cli.main(["bench", "--n", "100", "--dims", "a,b"]) != cli.EXIT_OK
    assert cli.main(["bench", "--dims", "8"]) == cli.EXIT_ARGUMENT


@pytest.mark.gpu
def test_accuracy_command_reproduces_reference_c1(tmp_path, golden_meta, capsys):
    """`accuracy --mode exact` at C1: the GPU FP64 truth (all 16384 points)
    and the exact kernel give the reference's own overlap; the saved-truth
    path (a pairs file + manifest of the same dataset) gives the same
    numbers; the histogram CSV has --bins rows."""
    c1 = golden_meta["C1"]
    ref = golden_meta.get("C1_accuracy")
    args = ["accuracy", "--synthetic", "16384x128", "--seed", "12345", "--epsilon",
            repr(c1["epsilon"]), "--json"]
    rc = cli.main(args + ["--mode", "exact", "--hist-out", str(tmp_path / "h.csv"),
                          "--bins", "21", "--manifest", str(tmp_path / "acc.json")])
    assert rc == 0
    out = {o["metric"]: o["value"] for o in
           (json.loads(x) for x in capsys.readouterr().out.strip().splitlines())}
    if ref is not None:
        assert out["pairs_truth"] == ref["truth_pairs"]
        assert abs(out["overlap"] - ref["overlap"]) < 1e-12
    assert out["pairs_mixed"] == c1["pairs"]
    lines = (tmp_path / "h.csv").read_text().strip().splitlines()
    assert lines[0] == "bin_lo,bin_hi,count" and len(lines) == 22
    assert sum(int(x.split(",")[2]) for x in lines[1:]) == out["matched_pairs"]
    # saved truth: write the FP64 truth as a pairs file + manifest, then reuse it
    from paper_2508_21230_b200 import accuracy
    ds = F.generate_synthetic(16384, 128, seed=12345)
    truth = accuracy.brute_force_fp64(ds, c1["epsilon"])
    cli.write_pairs(tmp_path / "t.pairs", truth)
    (tmp_path / "t.pairs.manifest.json").write_text(json.dumps(
        {"dataset": {"sha256": cli.dataset_sha256(ds)}, "epsilon": c1["epsilon"]}))
    rc = cli.main(args + ["--mode", "exact", "--truth-pairs", str(tmp_path / "t.pairs")])
    assert rc == 0
    out2 = {o["metric"]: o["value"] for o in
            (json.loads(x) for x in capsys.readouterr().out.strip().splitlines())}
    assert out2["overlap"] == out["overlap"] and out2["pairs_truth"] == out["pairs_truth"]
    # tcgen05 path on a row sample
    rc = cli.main(args + ["--sample-blocks", "8"])
    assert rc == 0
    out3 = {o["metric"]: o["value"] for o in
            (json.loads(x) for x in capsys.readouterr().out.strip().splitlines())}
    assert out3["sample_points"] == 1024 and out3["overlap"] > 0.99


@pytest.mark.gpu
def test_bench_command_sweep(tmp_path):
    """`bench` sweeps (|D|, d), writes the reference's CSV columns plus the
    kernel-only columns, and a manifest whose digests equal the join's."""
    import csv
    rc = cli.main(["bench", "--ns", "4096,8192", "--dims", "64,200", "--epsilon", "2.0",
                   "--repeats", "3", "--csv", str(tmp_path / "b.csv"),
                   "--manifest", str(tmp_path / "b.json")])
    assert rc == 0
    rows = list(csv.DictReader(open(tmp_path / "b.csv")))
    assert [(int(r["n"]), int(r["d"])) for r in rows] == [(4096, 64), (4096, 200),
                                                          (8192, 64), (8192, 200)]
    for r in rows:
        assert float(r["distance_tflops"]) > 0 and int(r["pairs"]) >= int(r["n"])
        assert "join_tc" in r["kernel"]
        assert int(r["d_padded"]) % 16 == 0
    man = json.loads((tmp_path / "b.json").read_text())
    assert len(man["runs"]) == 4
    ds = F.generate_synthetic(4096, 64, seed=12345)
    rs = F.self_join(F.to_half(ds), 2.0)
    import hashlib
    assert man["runs"][0]["result_sha256"] == hashlib.sha256(cli.pairs_payload(rs)).hexdigest()
