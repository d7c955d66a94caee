"""CLI front end on the device: `synthetic` writes the reference-format
table for a BASELINE configuration; `verify --fast` passes."""
import json

import pytest

from paper_2605_24514_b200 import cli

pytestmark = pytest.mark.gpu


def test_synthetic_config1(tmp_path):
    out = tmp_path / "cfg1"
    assert cli.main(["synthetic", "--config", "1", "--seed", "0", "--out", str(out),
                     "--events", "120"]) == cli.EXIT_OK
    lines = (out / "synthetic.csv").read_text().splitlines()
    assert len(lines) == 3 + 121  # header lines + init record + one per event
    man = json.loads((out / "manifest.json").read_text())
    assert man["config"]["k"] == 10 and man["seed"] == 0
    # the periodic policy refreshed at t = 100
    refreshed = [ln.split(",")[9] for ln in lines[3:]]
    assert refreshed[100] == "True"


def test_verify_fast():
    assert cli.main(["verify", "--fast"]) == cli.EXIT_OK
