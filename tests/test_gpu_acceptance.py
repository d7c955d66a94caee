"""The reference's externally guaranteed properties of the update path
(its acceptance checks 1, 2, 3, 4, 8 and 12, src/svdstream/acceptance.py),
restated against the GPU engine: each property is checked against a direct
recomputation from the tracked matrix, never against the incremental path
itself."""

import math

import numpy as np
import pytest

from paper_2605_24514_b200 import SvdEngine, compute_oracle, error_ratio, frob_error, full_svd
from paper_2605_24514_b200.linalg import frobenius_norm, orthonormality_defect, reconstruct

pytestmark = pytest.mark.gpu


def _low_rank(m, n, rank, noise, seed):
    rng = np.random.default_rng(seed)
    return rng.standard_normal((m, rank)) @ rng.standard_normal((rank, n)) + \
        noise * rng.standard_normal((m, n))


@pytest.mark.parametrize("kind", ["rows", "cols"])
def test_appends_exact_below_rank_budget(kind):
    """500 noise-free appends with k at twice the latent rank reconstruct
    the tracked matrix to 1e-8 max(1, ||A||_F) at every step (check 1)."""
    rng = np.random.default_rng(21)
    m, n, rank, k = 40, 30, 5, 10
    x = rng.standard_normal((m, rank))
    y = rng.standard_normal((n, rank))
    eng = SvdEngine(x @ y.T, k, capacity=(m + 520, n + 520, k))
    worst = 0.0
    for _ in range(500):
        if kind == "rows":
            eng.row_append(y @ rng.standard_normal(rank))
        else:
            m_now = eng.shape[0]
            x = np.vstack([x, rng.standard_normal((m_now - x.shape[0], rank))]) if m_now > x.shape[0] else x
            eng.col_append(x @ rng.standard_normal(rank))
        a = eng.tracked
        err = frobenius_norm(a - reconstruct(eng.factors))
        worst = max(worst, err / (1e-8 * max(1.0, math.sqrt(float(np.sum(a * a))))))
    assert worst <= 1.0


def test_rank_one_matches_projection_identity():
    """Rank-1 updates equal P_U (A_k + delta e_i e_j^T) P_V entrywise within
    1e-10 (check 2; engine.py:149-167, PAPER eq. for the projection rule)."""
    rng = np.random.default_rng(22)
    worst = 0.0
    for _ in range(40):
        eng = SvdEngine(rng.standard_normal((12, 3)) @ rng.standard_normal((3, 9)), 3)
        for _ in range(10):
            i, j = int(rng.integers(12)), int(rng.integers(9))
            delta = float(rng.normal())
            before = eng.factors
            approx = reconstruct(before)
            eng.rank_one_update(i, j, delta)
            pu = before.u @ before.u.T
            pv = before.vt.T @ before.vt
            target = approx + delta * np.outer(pu[:, i], pv[j, :])
            worst = max(worst, float(np.max(np.abs(reconstruct(eng.factors) - target))))
    assert worst <= 1e-10


def test_mixed_stream_orthonormal_and_optimality_floor():
    """A 4,000-event mixed stream (rows, columns, rank-1) with refresh every
    200 keeps both bases orthonormal to 1e-8 (check 3) and every error ratio
    >= 1 - 1e-9 (check 4); the tracked squared norm matches a direct
    recomputation to 1e-9 relative (check 8)."""
    rng = np.random.default_rng(23)
    m, n, rank, k = 60, 40, 6, 8
    eng = SvdEngine(_low_rank(m, n, rank, 0.05, 23), k, capacity=(m + 2100, n + 2100, k))
    worst_defect, ratios = 0.0, []
    for t in range(1, 4001):
        mm, nn = eng.shape
        kind = rng.integers(3)
        if kind == 0:
            eng.row_append(rng.standard_normal(nn))
        elif kind == 1 and nn < n + 300:
            eng.col_append(rng.standard_normal(mm))
        else:
            eng.rank_one_update(int(rng.integers(mm)), int(rng.integers(nn)), float(rng.normal(0, 0.1)))
        if t % 200 == 0:
            o = compute_oracle(eng, eng.work_rank)
            ratios.append(error_ratio(frob_error(eng), o.frob_opt))
            eng.refresh()
        if t % 100 == 0:
            f = eng.factors
            worst_defect = max(worst_defect, orthonormality_defect(f.u),
                               orthonormality_defect(f.vt.T))
    assert worst_defect <= 1e-8
    assert all(r >= 1.0 - 1e-9 for r in ratios if r == r)
    a = eng.tracked
    direct = float(np.sum(a * a))
    assert abs(eng.sq_norm - direct) <= 1e-9 * direct


def test_long_rank_one_stream_norm_tracking():
    """10,000 rank-1 updates: the N_t recurrence agrees with ||A||_F^2 to
    1e-9 relative and the bases stay orthonormal (checks 3 and 8)."""
    rng = np.random.default_rng(24)
    eng = SvdEngine(_low_rank(100, 50, 5, 0.1, 24), 5)
    for _ in range(10_000):
        eng.rank_one_update(int(rng.integers(100)), int(rng.integers(50)), float(rng.normal(0, 0.1)))
    a = eng.tracked
    direct = float(np.sum(a * a))
    assert abs(eng.sq_norm - direct) <= 1e-9 * direct
    f = eng.factors
    assert orthonormality_defect(f.u) <= 1e-8 and orthonormality_defect(f.vt.T) <= 1e-8


def test_batch_svd_matches_gram_eigenvalues():
    """Singular values of 200 random small matrices match sqrt of the Gram
    eigenvalues from an independent eigensolver within 1e-8 (check 12)."""
    rng = np.random.default_rng(12)
    worst = 0.0
    for _ in range(200):
        m, n = int(rng.integers(1, 13)), int(rng.integers(1, 11))
        a = rng.standard_normal((m, n))
        s = full_svd(a).s
        ref = np.sqrt(np.clip(np.linalg.eigvalsh(a.T @ a), 0.0, None))[::-1][: len(s)]
        worst = max(worst, float(np.max(np.abs(s - ref))))
    assert worst <= 1e-8
