"""The device benchmark harness and CLI (paper_2005_12648_b200.bench / .cli), mirroring
the reference's tests/test_bench.py and tests/test_cli.py.

CPU tests cover configuration, the size grammar, CSV round trips, the speedup table
and the median-quality arithmetic (with the oracle's Alg. 1 and a numpy optimal
search, pinned to the reference's own study output in tests/golden/bench.npz).
GPU tests run the CLI end to end: timing grid, validate-only and the study on device.
"""
import hashlib
import os

import numpy as np
import pytest

from oracle import oracle as orc
from paper_2005_12648_b200 import bench as hb
from paper_2005_12648_b200 import cli
from paper_2005_12648_b200.workloads import generate_input as gen_host

GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "bench.npz"))


def test_generator_matches_reference_digests():
    for (size, split, seed, eb, middle), digest in zip(GOLD["gen_params"], GOLD["gen_sha"]):
        keys, payload, m = gen_host(int(size), float(split), int(seed), int(eb))
        assert m == int(middle)
        h = hashlib.sha256(np.ascontiguousarray(keys).tobytes())
        h.update(np.ascontiguousarray(payload).tobytes())
        assert h.hexdigest() == str(digest), (size, split, seed, eb)


def _optimal_host(a, b):
    """numpy restatement of find_median_optimal (median.py:63-100) for the CPU tests."""
    la, lb = len(a), len(b)
    total = la + lb
    if la == 0:
        return 0, min(max(total // 2, 0), lb)
    lo = np.zeros(la + 1, np.int64)
    lo[1:] = np.searchsorted(b, a, side="left")
    hi = np.full(la + 1, lb, np.int64)
    hi[:la] = np.searchsorted(b, a, side="right")
    pa = np.arange(la + 1, dtype=np.int64)
    fl = np.clip((total - 2 * pa) // 2, lo, hi)
    ce = np.clip((total - 2 * pa + 1) // 2, lo, hi)
    bf, bc = np.abs(2 * (pa + fl) - total), np.abs(2 * (pa + ce) - total)
    pb = np.where(bc < bf, ce, fl)
    i = int(np.argmin(np.minimum(bf, bc)))
    return i, int(pb[i])


def test_quality_arithmetic_matches_reference_study():
    """largest_leaf_pair + the study's averaging reproduce the reference's rows exactly."""
    sizes, splits = [int(s) for s in GOLD["quality_sizes"]], [float(s) for s in GOLD["quality_splits"]]
    want = {(int(t), int(s)): v for t, s, v in GOLD["quality"]}
    med = lambda a, b: orc.find_median(np.ascontiguousarray(a), np.ascontiguousarray(b))  # noqa: E731
    for t in hb.QUALITY_THREADS:
        for size in sizes:
            diffs = []
            for split in splits:
                keys, _, middle = gen_host(size, split, 1)
                heur = hb.largest_leaf_pair(keys, middle, t, med)
                best = hb.largest_leaf_pair(keys, middle, t, _optimal_host)
                diffs.append(0.0 if best == 0 else (heur - best) / best)
            assert float(np.mean(diffs)) == want[(t, size)], (t, size)


def test_config_validation_errors():
    for bad in (dict(sizes=(-1,)), dict(elem_bytes=(3,)), dict(splits=(0.0,)), dict(splits=(1.0,)),
                dict(reps=0), dict(methods=("nope",)), dict(threads=(3,)), dict(splits=(0.501, 0.499)),
                dict(splits=(0.001,)), dict(device="cpu")):
        with pytest.raises(hb.ConfigError):
            hb.BenchConfig(**bad).validate()
    assert hb.BenchConfig(splits=(0.333,)).validate().splits == (0.33,)


def test_cells_and_threads():
    cfg = hb.BenchConfig(sizes=(4, 8), elem_bytes=(4, 1024), splits=(0.5,), threads=(2, 4),
                         methods=("seq-buffered", "srecpar-ls"), max_bytes=4096).validate()
    cells = list(hb.iter_cells(cfg))
    assert hb.threads_for("seq-buffered", cfg) == (1,) and hb.threads_for("soptmov", cfg) == (2, 4)
    # 1024-byte records of size 8 exceed max_bytes
    assert ("seq-buffered", 1, 1024, 8, 0.5) not in cells and ("seq-buffered", 1, 1024, 4, 0.5) in cells
    assert len(cells) == 3 + 2 * 3


def test_csv_round_trip(tmp_path):
    recs = [hb.BenchRecord("soptmov", 8, 64, 1024, 0.25, 10.5, 9.0, 12.25),
            hb.BenchRecord("seq-buffered", 1, 4, 16, 0.75, 1.0, 1.0, 1.0)]
    p = tmp_path / "r.csv"
    hb.write_records_csv(p, recs)
    assert p.read_text().splitlines()[0] == hb.RECORD_HEADER
    assert hb.read_records_csv(p) == recs
    (tmp_path / "bad.csv").write_text("x,y\n")
    with pytest.raises(hb.ConfigError):
        hb.read_records_csv(tmp_path / "bad.csv")
    q = tmp_path / "q.csv"
    hb.write_quality_csv(q, [hb.QualityRow(2, 16, 0.125)])
    assert q.read_text().splitlines() == [hb.QUALITY_HEADER, "2,16,0.125"]
    with pytest.raises(ValueError):
        hb.BenchRecord("soptmov", 8, 64, 1024, 0.25, 1.0, 2.0, 3.0)


def test_speedup_table():
    recs = [hb.BenchRecord("seq-buffered", 1, 4, 16, sp, m, m, m) for sp, m in ((0.25, 100.0), (0.75, 200.0))]
    recs += [hb.BenchRecord("soptmov", 8, 4, 16, sp, m, m, m) for sp, m in ((0.25, 50.0), (0.75, 50.0))]
    rows = hb.speedup_table(recs, "seq-buffered")
    assert rows[0] == hb.SpeedupRow("seq-buffered", 1, 4, 16, 1.0)
    assert rows[1] == hb.SpeedupRow("soptmov", 8, 4, 16, 3.0)
    with pytest.raises(hb.ConfigError):
        hb.speedup_table(recs, "srecpar-ls")
    with pytest.raises(hb.ConfigError):
        hb.speedup_table(recs + [hb.BenchRecord("soptmov", 8, 4, 32, 0.5, 1.0, 1.0, 1.0)], "seq-buffered")


def test_cli_parsing(capsys):
    assert cli.parse_count("2^10") == 1024 and cli.parse_count(" 17 ") == 17
    with pytest.raises(hb.ConfigError):
        cli.parse_count("3^2")
    assert cli.parse_sizes("2^2..2^5,100") == (4, 8, 16, 32, 100)
    for bad in ("", "8..4", "0..4"):
        with pytest.raises(hb.ConfigError):
            cli.parse_sizes(bad)
    assert cli.effective_threads((3, 4, 16, 17)) == (2, 4, 16)
    assert "rounding threads 3 down to 2" in capsys.readouterr().err


def test_cli_config_errors_exit_2(tmp_path):
    out = str(tmp_path / "x.csv")
    assert cli.main(["--elem-bytes", "2", "--out", out]) == cli.EXIT_CONFIG
    assert cli.main(["--device", "cpu", "--out", out]) == cli.EXIT_CONFIG
    assert cli.main(["--methods", "bogus", "--out", out]) == cli.EXIT_CONFIG
    assert not os.path.exists(out)


@pytest.mark.gpu
def test_cli_grid_on_device(tmp_path, capsys):
    out = tmp_path / "gpu.csv"
    rc = cli.main(["--sizes", "2^4..2^12", "--elem-bytes", "4,64,512", "--reps", "2", "--threads", "8",
                   "--out", str(out), "--speedup-baseline", "seq-buffered"])
    assert rc == cli.EXIT_OK
    recs = hb.read_records_csv(out)
    assert len(recs) == (2 + 3) * 3 * 9 * 3
    assert all(r.min_ns > 0 for r in recs)
    assert "speedup soptmov t=8" in capsys.readouterr().out
    assert cli.main(["--sizes", "2^12", "--elem-bytes", "16384,65540", "--validate-only",
                     "--out", str(tmp_path / "v.csv")]) == cli.EXIT_OK
    assert not (tmp_path / "v.csv").exists()


@pytest.mark.gpu
def test_cli_median_quality_on_device_matches_reference(tmp_path):
    sizes = ",".join(str(int(s)) for s in GOLD["quality_sizes"])
    out = tmp_path / "q.csv"
    assert cli.main(["--study", "median-quality", "--sizes", sizes, "--out", str(out)]) == cli.EXIT_OK
    got = np.loadtxt(out, delimiter=",", skiprows=1)
    assert np.array_equal(got, GOLD["quality"])
