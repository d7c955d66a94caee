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
