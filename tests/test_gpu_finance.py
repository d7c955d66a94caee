"""Config 3 per-tick risk on the device (finance.py:326-371 + BASELINE's
diagonal term and 99% VaR) against the host restatement on the same
factors, over the first ticks of the synthetic return panel."""

import numpy as np
import pytest

from oracle import OracleEngine, low_rank_covariance as o_cov, portfolio_vol as o_vol
from paper_2605_24514_b200 import SvdEngine, workloads
from paper_2605_24514_b200.finance import (Z99, PortfolioSpec, covariance_rel_error,
                                           equal_weights, low_rank_covariance, portfolio_vol,
                                           risk, risk_rel_error)

pytestmark = pytest.mark.gpu


def test_cfg3_risk_matches_host_restatement():
    a0, events, meta = workloads.cfg3(t_total=352)
    k = meta["k"]
    eng = SvdEngine(a0, k)
    ora = OracleEngine(a0, k)
    n = a0.shape[1]
    rng = np.random.default_rng(2)
    w2 = rng.uniform(0.0, 1.0, n)
    ports = [equal_weights(n), PortfolioSpec(w2 / w2.sum(), "random")]
    for t, (_, x) in enumerate(events[:60]):
        eng.row_append(x)
        ora.row_append(x)
        rows = eng.shape[0]
        rec = risk(eng, rows, ports)
        f = eng.factors
        cov_h = o_cov(f.s, f.vt, rows)
        np.testing.assert_allclose(rec.cov, cov_h, rtol=0, atol=1e-14 * np.abs(cov_h).max())
        assert np.array_equal(rec.cov, rec.cov.T)
        tracked = eng.tracked
        d_h = np.maximum(0.0, np.sum(tracked * tracked, axis=0) / (rows - 1) - np.diag(cov_h))
        np.testing.assert_allclose(rec.diag, d_h, rtol=0, atol=1e-13 * np.abs(cov_h).max())
        for p in ports:
            v = o_vol(cov_h, p.weights)
            assert abs(rec.vol_lr[p.label] - v) <= 1e-12 * v
            vd = np.sqrt(p.weights @ (cov_h + np.diag(d_h)) @ p.weights)
            assert abs(rec.vol_lr_diag[p.label] - vd) <= 1e-12 * vd
            assert abs(rec.var99[p.label] - Z99 * vd) <= 1e-12 * vd
        # incremental vs the oracle engine's covariance (trajectory parity)
        fo = ora.factors
        assert covariance_rel_error(rec.cov, o_cov(fo.s, fo.vt, rows)) < 1e-8
    # reference helper contracts
    c = low_rank_covariance(eng, eng.shape[0])
    assert portfolio_vol(c, ports[0]) > 0.0
    assert risk_rel_error(1.1, 1.0) == pytest.approx(0.1)
    with pytest.raises(ValueError):
        risk(eng, 1, ports)
    with pytest.raises(ValueError):
        PortfolioSpec(np.array([0.5, 0.6]), "bad")


class TestLowRankCovariance:
    """finance.py:326-335 on the device (ported from the reference's
    tests/test_finance.py TestLowRankCovariance)."""

    def test_two_day_single_asset(self):
        from paper_2605_24514_b200 import full_svd
        f = full_svd(np.array([[1.0], [-1.0]]))
        cov = low_rank_covariance(f, t=2)
        assert cov.shape == (1, 1)
        assert abs(cov[0, 0] - 2.0) < 1e-12

    def test_orthogonal_columns_give_diagonal(self):
        from paper_2605_24514_b200 import full_svd
        r = np.array([[1.0, 0.0], [0.0, 2.0], [-1.0, 0.0], [0.0, -2.0]])
        cov = low_rank_covariance(full_svd(r), t=4)
        assert abs(cov[0, 1]) < 1e-12 and abs(cov[1, 0]) < 1e-12

    def test_matches_gram_matrix(self):
        from paper_2605_24514_b200 import full_svd
        rng = np.random.default_rng(6)
        r = rng.standard_normal((50, 6))
        cov = low_rank_covariance(full_svd(r), t=50)
        assert np.allclose(cov, r.T @ r / 49.0, atol=1e-9)

    def test_symmetric(self):
        from paper_2605_24514_b200 import full_svd
        rng = np.random.default_rng(7)
        cov = low_rank_covariance(full_svd(rng.standard_normal((30, 5))), t=30)
        assert np.array_equal(cov, cov.T)

    def test_needs_two_rows(self):
        from paper_2605_24514_b200 import full_svd
        with pytest.raises(ValueError):
            low_rank_covariance(full_svd(np.ones((1, 2))), t=1)
