"""Per-tick portfolio risk of BASELINE config 3 (finance.py:266-371).

The covariance implied by the incremental factors, its diagonal correction
and the portfolio volatilities are computed on the device from the engine's
V, s and tracked returns (isvd_engine_risk, csrc/metrics.cu); the small
host helpers keep the reference's names, contracts and errors.

Reference quantities (finance.py:326-371): low_rank_covariance =
V diag(s^2) V^T / (t - 1) symmetrised; portfolio_vol = sqrt(w'Cw) with a
ValueError below -1e-10; covariance_rel_error; risk_rel_error.  BASELINE
config 3 also asks for the low-rank-plus-diagonal covariance and a 99%
Gaussian VaR, which the reference does not implement; they
are defined here as D = max(0, diag(sample cov) - diag(cov_lr)) over the
mean-centred returns and VaR99 = Phi^{-1}(0.99) * sqrt(w'(cov_lr + D)w).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import _lib
from .linalg import as_matrix, frobenius_norm

Z99 = 2.3263478740408408  # Phi^{-1}(0.99)


@dataclass
class PortfolioSpec:
    """Long-only weights over N assets, summing to one (finance.py:266-286)."""

    weights: np.ndarray
    label: str

    def __post_init__(self):
        w = np.asarray(self.weights, dtype=np.float64)
        if w.ndim != 1 or w.size < 1:
            raise ValueError(f"weights must be a nonempty 1-D array, got shape {w.shape}")
        if np.any(w < 0.0):
            raise ValueError(f"portfolio {self.label!r} has negative weights")
        if abs(float(w.sum()) - 1.0) > 1e-12:
            raise ValueError(f"portfolio {self.label!r} weights sum to {w.sum()!r}, expected 1")
        self.weights = w

    @property
    def n_assets(self) -> int:
        return self.weights.shape[0]


def equal_weights(n: int, label: str = "equal") -> PortfolioSpec:
    """The 1/N portfolio (finance.py:289-293)."""
    if n < 1:
        raise ValueError(f"need at least one asset, got {n}")
    return PortfolioSpec(np.full(n, 1.0 / n), label)


@dataclass
class RiskRecord:
    cov: np.ndarray          # (n, n) low-rank covariance
    diag: np.ndarray         # (n,) diagonal correction D
    vol_lr: dict             # label -> sqrt(w' cov w)        (reference portfolio_vol)
    vol_lr_diag: dict        # label -> sqrt(w' (cov + D) w)   (BASELINE)
    var99: dict              # label -> Z99 * vol_lr_diag      (BASELINE)


def risk(engine, t: int, portfolios, b: int = 0) -> RiskRecord:
    """All per-tick risk quantities of stream `b` in one device pass."""
    h = engine._h
    bsz, m, n, *_ = h.shape()
    ports = list(portfolios)
    for p in ports:
        if p.n_assets != n:
            raise ValueError(f"portfolio {p.label!r} has {p.n_assets} weights for a "
                             f"{n}-asset covariance")
    w = np.ascontiguousarray(np.stack([p.weights for p in ports]), dtype=np.float64)
    cov = np.empty((bsz, n, n))
    dg = np.empty((bsz, n))
    out = np.empty((bsz, len(ports), 4))
    _lib.check(h.lib.isvd_engine_risk(h.h, int(t), _lib.dptr(w), len(ports), _lib.dptr(cov),
                                      _lib.dptr(dg), _lib.dptr(out)))
    o = out[b]
    return RiskRecord(cov[b], dg[b], {p.label: float(o[i, 0]) for i, p in enumerate(ports)},
                      {p.label: float(o[i, 1]) for i, p in enumerate(ports)},
                      {p.label: float(o[i, 2]) for i, p in enumerate(ports)})


def low_rank_covariance(f, t: int) -> np.ndarray:
    """finance.py:326-335: V diag(s^2) V^T / (t - 1), symmetrised, on the
    device -- from an engine's factors (no host copy) or from SvdFactors."""
    if t < 2:
        raise ValueError(f"need at least 2 rows for a covariance, got t={t}")
    if hasattr(f, "_h"):
        n = f._h.shape()[2]
        return risk(f, t, [equal_weights(n)]).cov
    v = np.ascontiguousarray(np.asarray(f.vt, dtype=np.float64).T)
    s = np.ascontiguousarray(np.asarray(f.s, dtype=np.float64))
    n, r = v.shape
    cov = np.empty((n, n))
    _lib.check(_lib.load().isvd_low_rank_cov(n, r, _lib.dptr(v), _lib.dptr(s), int(t),
                                             _lib.dptr(cov)))
    return cov


def covariance_rel_error(inc, orc) -> float:
    """finance.py:338-347."""
    inc = as_matrix(inc, "incremental covariance")
    orc = as_matrix(orc, "baseline covariance")
    if inc.shape != orc.shape:
        raise ValueError(f"covariance shapes differ: {inc.shape} vs {orc.shape}")
    denom = frobenius_norm(orc)
    if denom <= 0.0:
        raise ValueError("baseline covariance has zero norm; relative error undefined")
    return frobenius_norm(inc - orc) / denom


def portfolio_vol(cov, portfolio: PortfolioSpec) -> float:
    """finance.py:350-364: sqrt(w'Cw), clamping tiny negatives."""
    cov = as_matrix(cov, "covariance")
    if cov.shape[0] != cov.shape[1]:
        raise ValueError(f"covariance must be square, got {cov.shape}")
    if portfolio.n_assets != cov.shape[0]:
        raise ValueError(f"portfolio {portfolio.label!r} has {portfolio.n_assets} weights "
                         f"for a {cov.shape[0]}-asset covariance")
    w = portfolio.weights
    quad = float(w @ cov @ w)
    if quad < -1e-10:
        raise ValueError(f"covariance is not PSD on {portfolio.label!r}: w'Cw = {quad}")
    return math.sqrt(max(0.0, quad))


def risk_rel_error(vol_inc: float, vol_orc: float) -> float:
    """finance.py:367-371."""
    if not vol_orc > 0.0:
        raise ValueError(f"baseline volatility must be positive, got {vol_orc}")
    return abs(vol_inc - vol_orc) / vol_orc


# --------------------------------------------------------------------------
# The returns-panel pipeline (finance.py:47-260 ingestion and panels,
# finance.py:374-521 the stream loop and its snapshots) on the device engine.

_FACTOR_VOLS = (0.012, 0.008, 0.005)  # finance.py:45-46
_IDIO_VOL = 0.004


@dataclass
class PriceTable:
    """Wide price panel: one row per date, one column per ticker (finance.py:52-67)."""

    dates: list
    tickers: list
    prices: np.ndarray

    def __post_init__(self):
        self.prices = as_matrix(self.prices, "prices")
        if self.prices.shape != (len(self.dates), len(self.tickers)):
            raise ValueError(f"prices shape {self.prices.shape} does not match "
                             f"{len(self.dates)} dates x {len(self.tickers)} tickers")


def log_returns(prices) -> np.ndarray:
    """finance.py:122-129: (T-1) x N log price ratios."""
    p = as_matrix(prices, "prices")
    if p.shape[0] < 2:
        raise ValueError(f"need at least 2 dates for returns, got {p.shape[0]}")
    if np.any(p <= 0.0):
        raise ValueError("prices must be strictly positive")
    return np.diff(np.log(p), axis=0)


def center_expanding(returns) -> np.ndarray:
    """finance.py:132-140: subtract the expanding mean (causal)."""
    r = as_matrix(returns, "returns")
    counts = np.arange(1, r.shape[0] + 1, dtype=np.float64)[:, None]
    return r - np.cumsum(r, axis=0) / counts


def center_ew(returns, alpha: float) -> np.ndarray:
    """finance.py:143-160: subtract an exponentially weighted mean (mu_0 = 0)."""
    alpha = float(alpha)
    if not 0.0 < alpha < 1.0:
        raise ValueError(f"alpha must be in (0, 1), got {alpha}")
    r = as_matrix(returns, "returns")
    centered = np.empty_like(r)
    mu = np.zeros(r.shape[1])
    for t in range(r.shape[0]):
        mu = (1.0 - alpha) * mu + alpha * r[t]
        centered[t] = r[t] - mu
    return centered


@dataclass
class ReturnsPanel:
    """Log returns plus their centered version, aligned on dates (finance.py:163-185)."""

    dates: list
    tickers: list
    returns: np.ndarray
    centered: np.ndarray
    centering_mode: str

    def __post_init__(self):
        self.returns = as_matrix(self.returns, "returns")
        self.centered = as_matrix(self.centered, "centered")
        expected = (len(self.dates), len(self.tickers))
        if self.returns.shape != expected or self.centered.shape != expected:
            raise ValueError(f"panel shapes {self.returns.shape}/{self.centered.shape} "
                             f"do not match {expected}")

    @property
    def shape(self):
        return self.returns.shape


def build_panel(table: PriceTable, centering: str = "expanding", alpha: float = 0.06):
    """finance.py:188-210."""
    r = log_returns(table.prices)
    if centering == "expanding":
        centered, mode = center_expanding(r), "expanding"
    elif centering == "ew":
        centered, mode = center_ew(r, alpha), f"exponentially_weighted(alpha={alpha:g})"
    else:
        raise ValueError(f"unknown centering {centering!r} (expected expanding|ew)")
    return ReturnsPanel(dates=table.dates[1:], tickers=table.tickers, returns=r,
                        centered=centered, centering_mode=mode)


def business_dates(start: str, periods: int) -> list:
    """ISO dates of `periods` business days from `start` (pandas bdate_range,
    as finance.py:252-255)."""
    import pandas as pd

    return [d.strftime("%Y-%m-%d") for d in pd.bdate_range(start, periods=periods)]


def gen_synthetic_panel(assets: int = 60, days: int = 1640, factors: int = 3, seed: int = 0,
                        regime_shift: int | None = None, shift_scale: float = 3.0) -> PriceTable:
    """finance.py:213-258: business-day prices from a latent factor model."""
    from .workloads import PANEL, substream

    if assets < 1:
        raise ValueError(f"assets must be >= 1, got {assets}")
    if days < 2:
        raise ValueError(f"days must be >= 2, got {days}")
    if factors < 1:
        raise ValueError(f"factors must be >= 1, got {factors}")
    n_ret = days - 1
    if regime_shift is not None and not 0 <= regime_shift < n_ret:
        raise ValueError(f"regime_shift must be in [0, {n_ret}), got {regime_shift}")
    vols = list(_FACTOR_VOLS[:factors])
    while len(vols) < factors:
        vols.append(vols[-1] * 0.7)
    rng = substream(seed, PANEL)
    loadings = rng.standard_normal((assets, factors))
    fac = rng.standard_normal((n_ret, factors)) * np.asarray(vols)
    idio = rng.standard_normal((n_ret, assets)) * _IDIO_VOL
    rets = fac @ loadings.T + idio
    if regime_shift is not None:
        rets[regime_shift:] *= float(shift_scale)
    base = rng.uniform(20.0, 200.0, assets)
    log_prices = np.vstack([np.zeros(assets), np.cumsum(rets, axis=0)])
    prices = base * np.exp(log_prices)
    return PriceTable(dates=business_dates("2017-01-02", days),
                      tickers=[f"A{i:03d}" for i in range(assets)], prices=prices)


def baseline_config3_panel(seed: int = 0) -> ReturnsPanel:
    """BASELINE config 3 as a ReturnsPanel: the seeded 2520 x 50 five-factor
    return panel of workloads.cfg3, full-sample mean-centred (the centred
    rows are both `returns` and `centered`), on business dates from
    2017-01-03."""
    from . import workloads

    _, _, meta = workloads.cfg3(seed)
    r = meta["panel"]
    return ReturnsPanel(dates=business_dates("2017-01-03", r.shape[0]),
                        tickers=[f"A{i:03d}" for i in range(r.shape[1])], returns=r,
                        centered=r, centering_mode="full_sample")


def dirichlet_portfolios(n: int, count: int, concentration: float = 1.0, seed: int = 0):
    """finance.py:296-312."""
    from .workloads import PORTFOLIO, substream

    if n < 1:
        raise ValueError(f"n must be >= 1, got {n}")
    if count < 1:
        raise ValueError(f"count must be >= 1, got {count}")
    if not concentration > 0.0:
        raise ValueError(f"concentration must be positive, got {concentration}")
    rng = substream(seed, PORTFOLIO)
    alpha = np.full(n, float(concentration))
    return [PortfolioSpec(rng.dirichlet(alpha), f"dirichlet{i + 1}") for i in range(count)]


@dataclass
class RiskSnapshot:
    """One logged day of the finance stream, post-refresh (finance.py:377-389),
    plus BASELINE config 3's low-rank-plus-diagonal volatility and 99% VaR
    of each portfolio (no reference counterpart)."""

    step: int
    date: str
    cov_rel_error: float
    risk_rel_error: dict
    angle_factor: float
    refreshed: bool
    rank: int
    update_time: float
    opt_time: float
    vol_lr_diag: dict | None = None
    var99: dict | None = None


def run_finance_stream(panel: ReturnsPanel, t0: int, k: int, policy=None, portfolios=None,
                       log_every: int = 5, tol: float = 1e-10,
                       reortho_guard: bool = False) -> list:
    """finance.py:392-475 on the device engine: rows appended one day at a
    time; at the logging cadence (and on the final day) a device batch SVD of
    the same rows and a snapshot of the post-refresh state."""
    import time

    from .engine import SvdEngine
    from .linalg import full_svd, principal_angle_max
    from .metrics import error_ratio, frob_error
    from .policies import (PolicyConfig, angle_should_refresh, error_should_refresh,
                           periodic_should_refresh)

    total, n = panel.shape
    if not 2 <= t0 < total:
        raise ValueError(f"t0 must be in [2, {total}), got {t0}")
    if not 1 <= k <= n:
        raise ValueError(f"k must be in [1, {n}], got {k}")
    if log_every < 1:
        raise ValueError(f"log_every must be >= 1, got {log_every}")
    policy = policy or PolicyConfig()
    portfolios = list(portfolios) if portfolios is not None else [equal_weights(n)]
    for p in portfolios:
        if p.n_assets != n:
            raise ValueError(f"portfolio {p.label!r} does not match {n} assets")
    returns = panel.centered
    engine = SvdEngine(returns[:t0], k, tol=tol, reortho_guard=reortho_guard)
    engine.set_reference()
    snapshots = []
    t_last = 0
    for day in range(t0, total):
        step = day - t0 + 1
        start = time.perf_counter()
        try:
            engine.row_append(returns[day])
        except ValueError as exc:
            raise ValueError(f"append failed on {panel.dates[day]}: {exc}") from exc
        engine.synchronize()
        update_time = time.perf_counter() - start
        rows = day + 1
        logged = step % log_every == 0 or day == total - 1
        batch, opt_time = None, 0.0
        if logged:
            start = time.perf_counter()
            batch = full_svd(returns[:rows])
            opt_time = time.perf_counter() - start
        fire = False
        if policy.kind == "periodic":
            fire = periodic_should_refresh(step, policy.period)
        elif policy.kind == "error" and batch is not None:
            width = engine.factors.rank
            e_opt = float(np.sqrt(np.sum(batch.s[width:] ** 2)))
            fire = error_should_refresh(error_ratio(frob_error(engine), e_opt), policy.gamma,
                                        step, t_last, policy.min_spacing)
        elif policy.kind == "angle" and batch is not None:
            width = engine.factors.rank
            fire = angle_should_refresh(principal_angle_max(engine.factors.u,
                                                            batch.u[:, :width]),
                                        policy.theta_max)
        if fire:
            engine.refresh(store_reference=True)
            t_last = step
        if logged:
            snapshots.append(_take_snapshot(engine, batch, rows, step, panel.dates[day],
                                            portfolios, fire, update_time, opt_time))
    return snapshots


def _take_snapshot(engine, batch, rows, step, date, portfolios, refreshed, update_time,
                   opt_time) -> RiskSnapshot:
    """finance.py:478-521 (covariances on the device)."""
    import logging

    from .linalg import SvdFactors, principal_angle_max

    inc = engine.factors
    width = inc.rank
    best = SvdFactors(np.ascontiguousarray(batch.u[:, :width]), batch.s[:width].copy(),
                      np.ascontiguousarray(batch.vt[:width, :]))
    angle = principal_angle_max(inc.vt.T, best.vt.T)
    cov_inc = low_rank_covariance(inc, rows)
    cov_best = low_rank_covariance(best, rows)
    cov_err = covariance_rel_error(cov_inc, cov_best)
    risks = {}
    for p in portfolios:
        vol_best = portfolio_vol(cov_best, p)
        try:
            risks[p.label] = risk_rel_error(portfolio_vol(cov_inc, p), vol_best)
        except ValueError:
            logging.getLogger(__name__).warning(
                "zero baseline volatility for %r on %s; error undefined", p.label, date)
            risks[p.label] = math.nan
    rr = risk(engine, rows, portfolios)
    return RiskSnapshot(step=step, date=date, cov_rel_error=cov_err, risk_rel_error=risks,
                        angle_factor=angle, refreshed=refreshed, rank=width,
                        update_time=update_time, opt_time=opt_time,
                        vol_lr_diag=rr.vol_lr_diag, var99=rr.var99)


def load_prices(path) -> PriceTable:
    """finance.py:70-119: read `date,<ticker>,...` (ISO dates, increasing,
    positive prices); days with a missing price are dropped."""
    import logging

    import pandas as pd

    try:
        df = pd.read_csv(path)
    except Exception as exc:  # pandas raises several parser types
        raise ValueError(f"could not parse price file {path}: {exc}") from exc
    if df.shape[1] < 2:
        raise ValueError(f"{path}: need a date column plus at least one ticker")
    if df.columns[0] != "date":
        raise ValueError(f"{path}: first column must be 'date', got {df.columns[0]!r}")
    tickers = [str(c) for c in df.columns[1:]]
    try:
        when = pd.to_datetime(df["date"], format="ISO8601")
    except (ValueError, TypeError) as exc:
        raise ValueError(f"{path}: unparseable date: {exc}") from exc
    for col in tickers:
        try:
            df[col] = pd.to_numeric(df[col])
        except (ValueError, TypeError) as exc:
            raise ValueError(f"{path}: column {col!r}: {exc}") from exc
    keep = ~df[tickers].isna().any(axis=1)
    dropped = int((~keep).sum())
    if dropped:
        logging.getLogger(__name__).info("%s: dropped %d day(s) with missing prices", path,
                                         dropped)
    when = when[keep]
    values = df.loc[keep, tickers].to_numpy(dtype=np.float64)
    if len(when) == 0:
        raise ValueError(f"{path}: no complete rows")
    dup = when.duplicated()
    if dup.any():
        raise ValueError(f"{path}: duplicate date {when[dup].iloc[0].date()}")
    if not when.is_monotonic_increasing:
        bad = int(np.argmax(np.diff(when.to_numpy()) < np.timedelta64(0)))
        raise ValueError(f"{path}: dates out of order at row {bad + 2}")
    nonpos = np.argwhere(values <= 0.0)
    if nonpos.size:
        r, c = nonpos[0]
        raise ValueError(f"{path}: nonpositive price {values[r, c]} for {tickers[c]} "
                         f"on {when.iloc[int(r)].date()}")
    return PriceTable(dates=[d.strftime("%Y-%m-%d") for d in when], tickers=tickers,
                      prices=values)
