"""File formats and the command line (reference
tensorio.py, geometry.py:194-303, cli.py), against files written by the
reference's own CLI (tests/golden/cli/, tests/golden/make_golden_cli.py)."""

import filecmp
import os
import re

import numpy as np
import pytest

from paper_2205_13542_b200 import cli
from paper_2205_13542_b200.errors import FileFormatError, ValidationError
from paper_2205_13542_b200.geometry import format_calibration, load_calibration, parse_calibration
from paper_2205_13542_b200.tensorio import deserialize_tensor, load_tensor, serialize_tensor

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = os.path.join(HERE, "golden", "cli")
FLAGS = ["--grid-extent", "8.0", "--cell-size", "0.5"]


def test_gen_workload_matches_reference_files(tmp_path):
    rc = cli.main(["gen-workload", "--cameras", "2", "--height", "4", "--width", "6",
                   "--depth-bins", "5", "--channels", "3", "--seed", "42", *FLAGS,
                   "--out-dir", str(tmp_path)])
    assert rc == 0
    for name in ("calibration.json", "features.bvpt", "logits.bvpt"):
        assert filecmp.cmp(tmp_path / name, os.path.join(GOLD, name), shallow=False), name


def test_tensor_round_trip_and_errors():
    a = np.arange(24, dtype=np.float32).reshape(2, 3, 4)
    blob = serialize_tensor(a)
    assert np.array_equal(deserialize_tensor(blob), a)
    with pytest.raises(FileFormatError, match="truncated"):
        deserialize_tensor(blob[:-3])
    with pytest.raises(FileFormatError, match="magic"):
        deserialize_tensor(b"XXXX" + blob[4:])
    with pytest.raises(FileFormatError, match="trailing"):
        deserialize_tensor(blob + b"\0")
    with pytest.raises(ValidationError):
        serialize_tensor(a.astype(np.float64))
    g = load_tensor(os.path.join(GOLD, "features.bvpt"))
    assert g.shape == (2, 3, 4, 6) and g.dtype == np.float32


def test_tensor_truncation_reports_the_field_being_read():
    """Every truncation of a BVPT blob names the field being read and its
    start offset, as the reference's take() does (tensorio.py:39-71): magic
    [0, 4), header [4, 8), shape[i] [8 + 4i, 12 + 4i), payload after."""
    a = np.arange(12, dtype=np.float32).reshape(3, 4)
    blob = serialize_tensor(a)
    fields = [(0, 4, "magic"), (4, 8, "header"), (8, 12, "shape[0]"), (12, 16, "shape[1]"),
              (16, len(blob), "payload")]
    for n in range(len(blob)):
        start, what = next((lo, w) for lo, hi, w in fields if lo <= n < hi)
        with pytest.raises(FileFormatError, match=rf"truncated while reading {re.escape(what)}") as ei:
            deserialize_tensor(blob[:n])
        assert ei.value.offset == start, (n, what)


def test_calibration_round_trip_and_field_errors():
    rig, spec = load_calibration(os.path.join(GOLD, "calibration.json"))
    with open(os.path.join(GOLD, "calibration.json")) as fh:
        assert format_calibration(rig, spec) + "\n" == fh.read()
    with pytest.raises(FileFormatError, match=r"cameras\[0\]\.fx"):
        parse_calibration('{"cameras": [{"fy": 1}], "frustum": {}}')
    with pytest.raises(FileFormatError, match="frustum"):
        parse_calibration('{"cameras": [{"id": 0, "fx": 1, "fy": 1, "cx": 0, "cy": 0, '
                          '"rotation": [1,0,0,0,1,0,0,0,1], "translation": [0,0,0]}]}')


def test_bad_input_exit_code(tmp_path, capsys):
    bad = tmp_path / "f.bvpt"
    bad.write_bytes(b"BVPT\x01")
    rc = cli.main(["pool", "--calib", os.path.join(GOLD, "calibration.json"), "--features",
                   str(bad), "--logits", str(bad), *FLAGS, "--out", str(tmp_path / "o.bvpt")])
    assert rc == 2
    assert "truncated" in capsys.readouterr().err


# ---- GPU: the CLI's pooling against the reference's files -----------------

def _pool_args(tmp_path, *extra):
    return ["pool", "--calib", os.path.join(GOLD, "calibration.json"),
            "--features", os.path.join(GOLD, "features.bvpt"),
            "--logits", os.path.join(GOLD, "logits.bvpt"), *FLAGS, *extra,
            "--out", str(tmp_path / "bev.bvpt")]


@pytest.mark.gpu
def test_cli_pool_exact_is_byte_identical(tmp_path):
    assert cli.main(_pool_args(tmp_path, "--exact")) == 0
    assert filecmp.cmp(tmp_path / "bev.bvpt", os.path.join(GOLD, "bev_interval.bvpt"),
                       shallow=False)


@pytest.mark.gpu
def test_cli_pool_fast_and_cached(tmp_path):
    assert cli.main(["cache-build", "--calib", os.path.join(GOLD, "calibration.json"), *FLAGS,
                     "--out", str(tmp_path / "cache.bvpc")]) == 0
    assert filecmp.cmp(tmp_path / "cache.bvpc", os.path.join(GOLD, "cache.bvpc"), shallow=False)
    assert cli.main(_pool_args(tmp_path, "--cache", os.path.join(GOLD, "cache.bvpc"))) == 0
    got = load_tensor(tmp_path / "bev.bvpt")
    want = load_tensor(os.path.join(GOLD, "bev_naive.bvpt"))
    assert np.abs(got - want).max() <= 1e-4 * max(1.0, float(np.abs(want).max()))


@pytest.mark.gpu
def test_cli_stale_cache_and_verify(tmp_path, capsys):
    rc = cli.main(["pool", "--calib", os.path.join(GOLD, "calibration.json"),
                   "--features", os.path.join(GOLD, "features.bvpt"),
                   "--logits", os.path.join(GOLD, "logits.bvpt"),
                   "--grid-extent", "8.0", "--cell-size", "0.25",
                   "--cache", os.path.join(GOLD, "cache.bvpc"), "--out", str(tmp_path / "o.bvpt")])
    assert rc == 2
    assert "stale" in capsys.readouterr().err
    small = ["--cameras", "2", "--height", "8", "--width", "12", "--depth-bins", "9",
             "--channels", "8", "--grid-extent", "16", "--cell-size", "0.5"]
    assert cli.main(["verify", *small]) == 0
    assert "PASS" in capsys.readouterr().out
    assert cli.main(["verify", *small, "--corrupt-backend", "interval"]) == 1
    assert "FAIL" in capsys.readouterr().out


@pytest.mark.gpu
def test_cli_pool_naive_is_byte_identical(tmp_path):
    """The reference CLI's `pool --backend naive` file (bev_naive.bvpt, made by
    the reference itself) is reproduced byte for byte."""
    assert cli.main(_pool_args(tmp_path, "--backend", "naive")) == 0
    assert filecmp.cmp(tmp_path / "bev.bvpt", os.path.join(GOLD, "bev_naive.bvpt"),
                       shallow=False)


@pytest.mark.gpu
def test_cli_bench_and_csv(tmp_path, capsys):
    """`bench` (reference cli.py:135-156): stage table and the reference's
    CSV columns; --sweep runs the three resolutions."""
    small = ["--cameras", "2", "--height", "8", "--width", "12", "--depth-bins", "9",
             "--channels", "8", "--grid-extent", "16", "--cell-size", "0.5"]
    csv_path = tmp_path / "bench.csv"
    assert cli.main(["bench", *small, "--reps", "2", "--warmups", "1", "--csv", str(csv_path)]) == 0
    out = capsys.readouterr().out
    assert "association_cold" in out and "association_cached" in out and "interval" in out
    lines = csv_path.read_text().splitlines()
    assert lines[0] == "backend,n_points,channels,stage,median_ms,min_ms,speedup_vs_baseline"
    stages = {ln.split(",")[3] for ln in lines[1:]}
    assert stages == {"association_cold", "association_cached", "pool"}
    assert cli.main(["bench", *small, "--reps", "1", "--warmups", "1", "--sweep",
                     "--backend", "interval"]) == 0
    assert capsys.readouterr().out.count("workload:") == 3
