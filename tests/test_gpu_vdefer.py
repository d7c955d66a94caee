"""Deferred right-basis rotation (isvd_engine_set_vdefer): rank-1 updates
rotate a small r x r G (V = V_base G) instead of V, the next row append
projects through G and folds it into its own V rotation.  It must reproduce
the eager engine and the oracle (reference restatement) on every mix of
events that can meet a pending G: runs of rank-1 updates, row appends,
column appends, reads of V (factors, metrics, risk), snapshot/restore,
refresh."""

import numpy as np
import pytest

from conftest import rel_err, sine_angle
from oracle import OracleEngine
from paper_2605_24514_b200 import BatchedSvdEngine, SvdEngine, frob_error, workloads

pytestmark = pytest.mark.gpu

SIGMA_RTOL = 1e-9
ANGLE_TOL = 1e-6


def _mixed_events(rng, t_total, m0, n0):
    """Runs of 1-3 rank-1 updates between appends; a column now and then."""
    ev, m, n = [], m0, n0
    for t in range(t_total):
        kind = t % 7
        if kind in (0, 4):
            ev.append(("row", rng.standard_normal(n)))
            m += 1
        elif kind == 6 and t % 21 == 6:
            ev.append(("col", rng.standard_normal(m)))
            n += 1
        else:
            ev.append(("r1", int(rng.integers(m)), int(rng.integers(n)), float(rng.normal(0, 0.3))))
    return ev


def _apply(e, ev):
    if ev[0] == "row":
        e.row_append(ev[1])
    elif ev[0] == "col":
        e.col_append(ev[1])
    else:
        e.rank_one_update(ev[1], ev[2], ev[3])


@pytest.mark.parametrize("k", [5, 17, 32])
@pytest.mark.parametrize("lazy_u", [True, False])
def test_vdefer_matches_eager_and_oracle(k, lazy_u):
    rng = np.random.default_rng(100 + k)
    m0, n0 = 90, 50
    a0 = rng.standard_normal((m0, n0)) @ np.diag(np.logspace(0, -2, n0)) @ rng.standard_normal((n0, n0))
    dfr, eag, cpu = SvdEngine(a0, k), SvdEngine(a0, k), OracleEngine(a0, k)
    dfr.set_vdefer(2)
    eag.set_vdefer(0)
    for e in (dfr, eag):
        e.set_lazy(lazy_u)
    events = _mixed_events(rng, 160, m0, n0)
    for t, ev in enumerate(events):
        for e in (dfr, eag, cpu):
            _apply(e, ev)
        if t % 29 == 3:  # reads of V in the middle of a pending G
            assert abs(frob_error(dfr) - frob_error(eag)) <= 1e-9 * max(1.0, frob_error(eag))
    fd, fe, fc = dfr.factors, eag.factors, cpu.factors
    assert rel_err(fd.s, fe.s) < 1e-11
    np.testing.assert_allclose(fd.vt, fe.vt, atol=1e-9)
    np.testing.assert_allclose(fd.u, fe.u, atol=1e-9)
    assert rel_err(fd.s, fc.s) < SIGMA_RTOL
    assert sine_angle(fd.u, fc.u) < ANGLE_TOL
    assert sine_angle(fd.vt.T, fc.vt.T) < ANGLE_TOL
    du, dv = dfr.ortho_defects()
    assert du < 1e-10 and dv < 1e-10


def test_vdefer_long_rank_one_run_then_row():
    """Fifty rank-1 updates accumulate in G, then one row append folds it."""
    rng = np.random.default_rng(7)
    a0 = rng.standard_normal((60, 8)) @ rng.standard_normal((8, 40)) + 0.01 * rng.standard_normal((60, 40))
    dfr, cpu = SvdEngine(a0, 8), OracleEngine(a0, 8)
    dfr.set_vdefer(2)
    for _ in range(50):
        i, j, d = int(rng.integers(60)), int(rng.integers(40)), float(rng.normal(0, 0.1))
        dfr.rank_one_update(i, j, d)
        cpu.rank_one_update(i, j, d)
    x = rng.standard_normal(40)
    dfr.row_append(x)
    cpu.row_append(x)
    fd, fc = dfr.factors, cpu.factors
    assert rel_err(fd.s, fc.s) < SIGMA_RTOL
    np.testing.assert_allclose(fd.u, fc.u, atol=1e-8)
    np.testing.assert_allclose(fd.vt, fc.vt, atol=1e-8)
    assert abs(dfr.sq_norm - cpu.sq_norm) <= 1e-12 * cpu.sq_norm


def test_vdefer_batched_auto_matches_off():
    """B = 64 turns deferral on by default; the same ticks with it off give
    the same factors per stream, and stream b matches the oracle."""
    B, T = 64, 40
    a0, ticks, streams = workloads.cfg5a_batch(5, B, m=96, n=48, rank=6, n_events=T)
    on, off = BatchedSvdEngine(a0, 6, m_cap=96 + T), BatchedSvdEngine(a0, 6, m_cap=96 + T)
    off.set_vdefer(0)
    for tk in ticks:
        for e in (on, off):
            if tk[0] == "row":
                e.row_append(tk[1])
            else:
                e.rank_one_update(tk[1], tk[2], tk[3])
    for b in (0, 17, 63):
        f1, f0 = on.factors(b), off.factors(b)
        assert rel_err(f1.s, f0.s) < 1e-11
        np.testing.assert_allclose(f1.vt, f0.vt, atol=1e-9)
        oe = OracleEngine(streams[b][0], 6)
        for e in streams[b][1]:
            if e[0] == "row":
                oe.row_append(e[1])
            else:
                oe.rank_one_update(e[1], e[2], e[3])
        assert rel_err(f1.s, oe.factors.s) < SIGMA_RTOL
        assert sine_angle(f1.vt.T, oe.factors.vt.T) < ANGLE_TOL


def test_vdefer_snapshot_restore_refresh():
    """A snapshot taken with G pending captures the materialised V; restore
    drops the pending G; refresh re-factors from the tracked matrix."""
    rng = np.random.default_rng(9)
    a0 = rng.standard_normal((70, 30))
    eng = BatchedSvdEngine(a0[None], 6, m_cap=80)
    eng.set_vdefer(2)
    eng.rank_one_update([3], [4], [0.5])
    eng.snapshot()
    ref = eng.factors(0)
    for _ in range(3):
        eng.rank_one_update([int(rng.integers(70))], [int(rng.integers(30))], [0.2])
    eng.restore()
    f = eng.factors(0)
    np.testing.assert_array_equal(f.vt, ref.vt)
    np.testing.assert_array_equal(f.s, ref.s)
    eng.rank_one_update([1], [2], [0.3])
    eng.refresh()
    eng.rank_one_update([5], [6], [-0.3])
    x = rng.standard_normal(30)
    eng.row_append(x[None])
    cpu = OracleEngine(a0, 6)
    cpu.rank_one_update(3, 4, 0.5)
    cpu.rank_one_update(1, 2, 0.3)
    cpu.refresh()
    cpu.rank_one_update(5, 6, -0.3)
    cpu.row_append(x)
    f = eng.factors(0)
    assert rel_err(f.s, cpu.factors.s) < SIGMA_RTOL
    assert sine_angle(f.vt.T, cpu.factors.vt.T) < ANGLE_TOL
    np.testing.assert_allclose(eng.tracked(0), cpu.tracked, atol=1e-12)


def test_vdefer_risk_reads_materialised_basis():
    """The device risk pass (low-rank covariance from V, s) right after a
    rank-1 update sees the folded V."""
    from paper_2605_24514_b200.finance import equal_weights, risk

    rng = np.random.default_rng(13)
    a0 = rng.standard_normal((80, 6)) @ rng.standard_normal((6, 20)) + 0.1 * rng.standard_normal((80, 20))
    on, off = SvdEngine(a0, 6), SvdEngine(a0, 6)
    on.set_vdefer(2)
    off.set_vdefer(0)
    for e in (on, off):
        e.rank_one_update(7, 3, 0.4)
        e.rank_one_update(2, 11, -0.2)
    r_on, r_off = risk(on, 80, [equal_weights(20)]), risk(off, 80, [equal_weights(20)])
    np.testing.assert_allclose(r_on.cov, r_off.cov, atol=1e-12)


@pytest.mark.parametrize("lazy_u", [True, False])
def test_deferred_rows_with_exact_zero_sigma(lazy_u):
    """Full-rank row appends keep V deferred (V_eff = [V | Z^T] G); when a
    tick leaves an exact zero singular value the completion first
    materialises that stream's V (tick.cu vdefer_materialise).  A rank-3
    start with k = 5 and in-span rows keeps sigma_4 = sigma_5 = 0 on every
    tick: the result must match the eager engine's live subspace and stay
    orthonormal through several deferral windows."""
    rng = np.random.default_rng(11)
    B, m0, n0, k = 64, 40, 30, 5
    a0 = rng.standard_normal((B, m0, 3)) @ rng.standard_normal((B, 3, n0))
    dfr, eag = BatchedSvdEngine(a0, k), BatchedSvdEngine(a0, k)
    dfr.set_vdefer(2)
    eag.set_vdefer(0)
    for e in (dfr, eag):
        e.set_lazy(lazy_u)
    basis = np.stack([eag.factors(b).vt[:3] for b in range(B)])
    cpu = OracleEngine(a0[9], k)
    for t in range(20):
        xs = np.einsum("bi,bij->bj", rng.standard_normal((B, 3)), basis)
        for e in (dfr, eag):
            e.row_append(xs)
        cpu.row_append(xs[9])
        if t % 7 == 6:
            ii = rng.integers(0, m0, B)
            jj = rng.integers(0, n0, B)
            for e in (dfr, eag):
                e.rank_one_update(ii, jj, np.zeros(B))
            cpu.rank_one_update(int(ii[9]), int(jj[9]), 0.0)
    for b in (0, 9, 63):
        fd, fe = dfr.factors(b), eag.factors(b)
        assert fd.s[3] == 0.0 and fd.s[4] == 0.0
        assert rel_err(fd.s[:3], fe.s[:3]) < 1e-11
        assert sine_angle(fd.vt[:3].T, fe.vt[:3].T) < 1e-9
        assert np.max(np.abs(fd.vt @ fd.vt.T - np.eye(k))) < 1e-10
        assert np.max(np.abs(fd.u.T @ fd.u - np.eye(k))) < 1e-10
    fc = cpu.factors
    assert rel_err(dfr.factors(9).s[:3], fc.s[:3]) < SIGMA_RTOL
    assert sine_angle(dfr.factors(9).vt[:3].T, fc.vt[:3].T) < ANGLE_TOL
