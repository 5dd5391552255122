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
