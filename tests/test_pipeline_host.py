"""Host side of the record formats and stream generators (CPU only): the
restated reference generators (workloads.py, finance.py) reproduce the
reference's streams and panels (checksums in tests/golden/ref_generators.json,
made by tests/golden/make_golden_pipeline.py from the real reference), the
finance/synthetic writers emit the reference's headers, price-file
validation follows finance.py:70-119, and CLI usage errors exit 2."""
import json

import numpy as np
import pytest

from conftest import GOLDEN_DIR, read_table
from paper_2605_24514_b200 import cli, finance, workloads

GEN = json.loads((GOLDEN_DIR / "ref_generators.json").read_text())


@pytest.mark.parametrize("scenario", ["rank1", "rows", "cols", "mixed"])
def test_stream_generators_match_reference(scenario):
    ev = workloads.build_events(workloads.StreamSpec(seed=7, scenario=scenario, events=300))
    acc = 0.0
    for e in ev:
        if e[0] == "rank1":
            acc += e[1] * 1e-3 + e[2] * 1e-6 + e[3]
        else:
            acc += float(np.sum(e[1] * np.arange(1, e[1].size + 1)))
    assert len(ev) == GEN[scenario]["count"]
    assert acc == GEN[scenario]["checksum"]


def test_low_rank_and_panel_generators_match_reference():
    a0 = workloads.gen_low_rank(50, 40, 5, 0.05, 7)
    assert float(np.sum(a0 * np.arange(1, 41))) == GEN["gen_low_rank_50x40_r5_seed7"]
    tab = finance.gen_synthetic_panel(assets=60, days=1640, factors=3, seed=2)
    assert float(np.sum(tab.prices)) == GEN["synthetic_panel_seed2"]
    assert [tab.dates[0], tab.dates[-1]] == GEN["panel_dates"]
    w = finance.dirichlet_portfolios(60, 2, 1.0, 2)
    assert [float(np.sum(p.weights * np.arange(1, 61))) for p in w] == GEN["dirichlet_seed2"]


def test_panel_construction():
    tab = finance.gen_synthetic_panel(assets=4, days=30, factors=2, seed=1)
    p = finance.build_panel(tab)
    assert p.shape == (29, 4) and p.dates == tab.dates[1:]
    np.testing.assert_allclose(p.centered[0], 0.0, atol=1e-18)  # first expanding-centred row
    np.testing.assert_allclose(p.centered, finance.center_expanding(p.returns))
    ew = finance.build_panel(tab, centering="ew", alpha=0.1)
    assert ew.centering_mode.startswith("exponentially_weighted")
    with pytest.raises(ValueError):
        finance.build_panel(tab, centering="median")
    cfg3 = finance.baseline_config3_panel(0)
    assert cfg3.shape == (2520, 50)
    np.testing.assert_allclose(cfg3.centered.mean(axis=0), 0.0, atol=1e-15)


def test_snapshot_writer_matches_reference_header(tmp_path):
    head, cols, rows = read_table(GOLDEN_DIR / "ref_finance_cfg3.csv.gz")
    snap = finance.RiskSnapshot(step=1, date="2017-12-29", cov_rel_error=0.5,
                                risk_rel_error={"equal": 0.1, "dirichlet1": 0.2, "dirichlet2": 0.3},
                                angle_factor=0.01, refreshed=False, rank=5, update_time=0.0,
                                opt_time=0.0)
    out = tmp_path / "finance.csv"
    cli.write_snapshots_csv(out, [snap], ["equal", "dirichlet1", "dirichlet2"],
                            "finance_manifest.json")
    h2, c2, r2 = read_table(out)
    assert h2 == head and c2 == cols
    assert r2[0][cols.index("refreshed")] == "False" and r2[0][cols.index("rank")] == "5"


def test_load_prices_validation(tmp_path):
    good = tmp_path / "p.csv"
    good.write_text("date,A,B\n2020-01-02,10,20\n2020-01-03,11,\n2020-01-06,12,21\n")
    tab = finance.load_prices(good)
    assert tab.dates == ["2020-01-02", "2020-01-06"] and tab.prices.shape == (2, 2)
    for text, msg in (("day,A\n2020-01-02,1\n", "first column"),
                      ("date,A\n2020-01-03,1\n2020-01-02,2\n", "out of order"),
                      ("date,A\n2020-01-02,1\n2020-01-02,2\n", "duplicate"),
                      ("date,A\n2020-01-02,1\n2020-01-03,-2\n", "nonpositive")):
        bad = tmp_path / "bad.csv"
        bad.write_text(text)
        with pytest.raises(ValueError, match=msg):
            finance.load_prices(bad)


def test_cli_usage_errors():
    assert cli.main(["synthetic", "--seed", "0", "--policy", "periodic"]) == cli.EXIT_USAGE
    assert cli.main(["finance", "--seed", "0"]) == cli.EXIT_USAGE  # no panel source
    assert cli.main(["finance", "--seed", "0", "--synthetic-panel", "--grid-k", "3"]) == \
        cli.EXIT_USAGE
