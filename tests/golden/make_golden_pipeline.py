"""Golden files for the record formats and the acceptance suite, made by the
REAL reference (run here only; the GPU box never needs /root/reference):

    python tests/golden/make_golden_pipeline.py

* ref_finance_cfg3.csv.gz -- BASELINE config 3 (the seeded 2520 x 50 panel of
  workloads.cfg3, t0 = 252, k = 5, angle refresh at 5 deg, equal-weight and
  two Dirichlet portfolios, a snapshot every day) through the reference's
  run_finance_stream, written by its write_snapshots_csv (cli.py:78-92).
* ref_finance_panel.csv.gz -- the reference's own synthetic price panel
  (gen_synthetic_panel, 60 assets, 1640 days, seed 2, expanding centering)
  with periodic refresh every 20 days, snapshots every 5 (the acceptance
  suite's refresh-20 run, acceptance.py:137-157).
* ref_synthetic_rank1.csv.gz -- `svdstream synthetic --seed 7 --scenario
  rank1 --events 2000 --refresh-every 500` records (write_records_csv).
* ref_generators.json -- checksums of the reference's stream generators.
* ref_acceptance.json -- run_acceptance(fast=False): number, name, passed,
  detail of every check.
"""
from __future__ import annotations

import gzip
import json
import shutil
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REPO = HERE.parent.parent
sys.path.insert(0, str(REPO))
sys.path.insert(0, str(HERE))

from make_golden import _import_reference  # noqa: E402
from paper_2605_24514_b200 import workloads  # noqa: E402


def _gz(src: Path, dst: Path):
    with open(src, "rb") as f, open(dst, "wb") as raw, gzip.GzipFile(fileobj=raw, mode="wb", mtime=0) as g:
        shutil.copyfileobj(f, g)


def main():
    _import_reference()
    from svdstream import acceptance, cli, finance, stream
    from svdstream.policies import PolicyConfig

    tmp = Path(tempfile.mkdtemp(prefix="svdstream_golden_"))
    # ---- config 3 through the reference's finance loop
    _, _, meta = workloads.cfg3(0)
    r = meta["panel"]
    import pandas as pd

    dates = [d.strftime("%Y-%m-%d") for d in pd.bdate_range("2017-01-03", periods=r.shape[0])]
    panel = finance.ReturnsPanel(dates=dates, tickers=[f"A{i:03d}" for i in range(r.shape[1])],
                                 returns=r, centered=r, centering_mode="full_sample")
    ports = [finance.equal_weights(r.shape[1])] + finance.dirichlet_portfolios(r.shape[1], 2, 1.0, 0)
    t0 = time.time()
    snaps = finance.run_finance_stream(panel, t0=252, k=5,
                                       policy=PolicyConfig(kind="angle",
                                                           theta_max=float(np.deg2rad(5.0))),
                                       portfolios=ports, log_every=1)
    cli.write_snapshots_csv(tmp / "finance.csv", snaps, [p.label for p in ports],
                            "finance_manifest.json")
    _gz(tmp / "finance.csv", HERE / "ref_finance_cfg3.csv.gz")
    print(f"cfg3 finance: {len(snaps)} snapshots, {sum(s.refreshed for s in snaps)} refreshes "
          f"({time.time() - t0:.1f}s)")
    # ---- the reference's synthetic price panel, refresh every 20
    p2 = finance.build_panel(finance.gen_synthetic_panel(assets=60, days=1640, factors=3, seed=2))
    ports2 = [finance.equal_weights(60)] + finance.dirichlet_portfolios(60, 1, 1.0, 2)
    snaps2 = finance.run_finance_stream(p2, t0=250, k=5,
                                        policy=PolicyConfig(kind="periodic", period=20),
                                        portfolios=ports2, log_every=5)
    cli.write_snapshots_csv(tmp / "panel.csv", snaps2, [p.label for p in ports2],
                            "finance_manifest.json")
    _gz(tmp / "panel.csv", HERE / "ref_finance_panel.csv.gz")
    print(f"panel finance: {len(snaps2)} snapshots")
    # ---- a synthetic run through the reference CLI's writer
    spec = stream.StreamSpec(seed=7, scenario="rank1", events=2000,
                             policy=PolicyConfig(kind="periodic", period=500), log_every=50)
    recs = stream.run_simulation(spec)
    cli.write_records_csv(tmp / "syn.csv", recs, "synthetic_rank1_manifest.json")
    _gz(tmp / "syn.csv", HERE / "ref_synthetic_rank1.csv.gz")
    # ---- generator checksums
    gens = {}
    for sc in ("rank1", "rows", "cols", "mixed"):
        sp = stream.StreamSpec(seed=7, scenario=sc, events=300)
        ev = stream.build_events(sp)
        acc = 0.0
        for e in ev:
            if isinstance(e, stream.RankOneUpdate):
                acc += e.i * 1e-3 + e.j * 1e-6 + e.delta
            else:
                acc += float(np.sum(e.values * np.arange(1, e.values.size + 1)))
        gens[sc] = {"count": len(ev), "checksum": acc}
    a0 = stream.gen_low_rank(50, 40, 5, 0.05, 7)
    gens["gen_low_rank_50x40_r5_seed7"] = float(np.sum(a0 * np.arange(1, 41)))
    tab = finance.gen_synthetic_panel(assets=60, days=1640, factors=3, seed=2)
    gens["synthetic_panel_seed2"] = float(np.sum(tab.prices))
    gens["panel_dates"] = [tab.dates[0], tab.dates[-1]]
    w = finance.dirichlet_portfolios(60, 2, 1.0, 2)
    gens["dirichlet_seed2"] = [float(np.sum(p.weights * np.arange(1, 61))) for p in w]
    (HERE / "ref_generators.json").write_text(json.dumps(gens, indent=1) + "\n")
    # ---- the acceptance suite
    t0 = time.time()
    res = acceptance.run_acceptance(fast=False)
    out = [{"number": x.number, "name": x.name, "passed": x.passed, "detail": x.detail}
           for x in res]
    (HERE / "ref_acceptance.json").write_text(json.dumps(out, indent=1) + "\n")
    print(f"acceptance: {sum(x.passed for x in res)}/{len(res)} ({time.time() - t0:.0f}s)")
    for x in out:
        print(" ", x)


if __name__ == "__main__":
    main()
