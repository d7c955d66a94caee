"""Host-side risk helpers of config 3 (ported from the reference's
tests/test_finance.py TestPortfolios / TestCovarianceRelError /
TestPortfolioVol / test_risk_rel_error; finance.py:266-371)."""

import math

import numpy as np
import pytest

from paper_2605_24514_b200.finance import (PortfolioSpec, covariance_rel_error, equal_weights,
                                           portfolio_vol, risk_rel_error)


class TestPortfolios:
    def test_equal_weights(self):
        spec = equal_weights(4)
        assert np.allclose(spec.weights, 0.25, atol=1e-15)
        assert spec.label == "equal"

    def test_weights_must_sum_to_one(self):
        with pytest.raises(ValueError):
            PortfolioSpec(weights=np.array([0.5, 0.4]), label="short")

    def test_weights_must_be_nonnegative(self):
        with pytest.raises(ValueError):
            PortfolioSpec(weights=np.array([1.5, -0.5]), label="levered")

    def test_nonempty_one_dimensional(self):
        with pytest.raises(ValueError):
            PortfolioSpec(weights=np.ones((2, 2)) / 4, label="matrix")
        with pytest.raises(ValueError):
            equal_weights(0)


class TestCovarianceRelError:
    def test_identical_matrices(self):
        cov = np.eye(3)
        assert covariance_rel_error(cov, cov) == 0.0

    def test_one_percent_scale(self):
        cov = np.diag([2.0, 1.0])
        assert abs(covariance_rel_error(1.01 * cov, cov) - 0.01) < 1e-12

    def test_zero_baseline_rejected(self):
        with pytest.raises(ValueError):
            covariance_rel_error(np.eye(2), np.zeros((2, 2)))

    def test_shape_mismatch_rejected(self):
        with pytest.raises(ValueError):
            covariance_rel_error(np.eye(2), np.eye(3))


class TestPortfolioVol:
    def test_identity_covariance(self):
        vol = portfolio_vol(np.eye(2), equal_weights(2))
        assert abs(vol - math.sqrt(0.5)) < 1e-12

    def test_zero_covariance(self):
        assert portfolio_vol(np.zeros((3, 3)), equal_weights(3)) == 0.0

    def test_diagonal_covariance(self):
        spec = PortfolioSpec(weights=np.array([1.0, 0.0]), label="first")
        assert abs(portfolio_vol(np.diag([0.04, 0.01]), spec) - 0.2) < 1e-12

    def test_dimension_mismatch_rejected(self):
        with pytest.raises(ValueError):
            portfolio_vol(np.eye(3), equal_weights(2))

    def test_indefinite_quadratic_rejected(self):
        spec = PortfolioSpec(weights=np.array([1.0]), label="solo")
        with pytest.raises(ValueError):
            portfolio_vol(np.array([[-1.0]]), spec)

    def test_permutation_invariant(self):
        rng = np.random.default_rng(8)
        a = rng.standard_normal((6, 4))
        cov = a.T @ a
        w = rng.uniform(0.1, 1.0, 4)
        spec = PortfolioSpec(weights=w / w.sum(), label="w")
        perm = np.array([2, 0, 3, 1])
        permuted = PortfolioSpec(weights=spec.weights[perm], label="permuted")
        assert abs(portfolio_vol(cov, spec) - portfolio_vol(cov[np.ix_(perm, perm)], permuted)) < 1e-12


def test_risk_rel_error():
    assert risk_rel_error(1.0, 1.0) == 0.0
    assert abs(risk_rel_error(1.001, 1.0) - 0.001) < 1e-12
    with pytest.raises(ValueError):
        risk_rel_error(1.0, 0.0)
