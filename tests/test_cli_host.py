"""CLI front end (paper_2605_24514_b200/cli.py, after the reference's cli.py):
argument handling and the CSV table format on CPU; the device runs are in
tests/test_gpu_cli.py."""
from pathlib import Path

import pytest

from paper_2605_24514_b200 import cli
from paper_2605_24514_b200.metrics import MetricsRecord


def test_usage_errors_exit_2():
    assert cli.main(["synthetic", "--config", "9", "--seed", "0", "--out", "x"]) == cli.EXIT_USAGE
    assert cli.main([]) == cli.EXIT_USAGE


def test_csv_format(tmp_path: Path):
    recs = [MetricsRecord(step=0, frob_error=1.5, evr=0.9, rank=3, refreshed=False,
                          update_time=0.1, frob_opt=None, frob_gap=float("nan"))]
    p = tmp_path / "synthetic_rank1.csv"
    cli.write_records_csv(p, recs, "synthetic_rank1_manifest.json")
    lines = p.read_text().splitlines()
    assert lines[0] == "# manifest: synthetic_rank1_manifest.json"
    assert lines[1] == "# nondeterministic columns: update_time,opt_time"
    assert lines[2].split(",") == list(cli.SYNTHETIC_COLUMNS)
    row = dict(zip(cli.SYNTHETIC_COLUMNS, lines[3].split(",")))
    assert row["step"] == "0" and row["frob_error"] == "1.5" and row["frob_opt"] == "NaN"
    assert row["frob_gap"] == "NaN" and row["refreshed"] == "False" and row["rank"] == "3"
