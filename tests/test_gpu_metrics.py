"""Metrics, dense SVD and the simulation loop on the GPU (ported from the
reference's tests/test_metrics.py, test_linalg.py and test_stream.py)."""

import math

import numpy as np
import pytest

from conftest import rel_err, sine_angle
from oracle import full_svd as o_full_svd
from paper_2605_24514_b200 import (PolicyConfig, AdaptiveRankConfig, SvdEngine, compute_oracle,
                                   error_ratio, evr, frob_error, full_svd, is_defined,
                                   oracle_baseline, run_stream, truncated_svd)
from paper_2605_24514_b200.linalg import orthonormality_defect, reconstruct, frobenius_norm
from paper_2605_24514_b200.metrics import MetricsRecord, angle_to_opt, angle_to_ref, collect
from paper_2605_24514_b200 import workloads

pytestmark = pytest.mark.gpu


class TestDenseSvd:
    @pytest.mark.parametrize("m, n", [(1, 1), (2, 2), (3, 2), (2, 3), (8, 6), (6, 8), (12, 9),
                                      (40, 17), (17, 40), (200, 100), (100, 300), (333, 65)])
    def test_matches_lapack(self, m, n):
        rng = np.random.default_rng(m * 1000 + n)
        a = rng.standard_normal((m, n))
        f, fo = full_svd(a), o_full_svd(a)
        assert rel_err(f.s, fo.s) < 1e-12
        # SPEC.md full_svd post-condition: ||A - U S Vt||_F <= 1e-9 max(1, ||A||_F)
        assert frobenius_norm(a - reconstruct(f)) <= 1e-11 * max(1.0, frobenius_norm(a))
        # SPEC invariant is 1e-8; the accumulated Jacobi rotations sit ~1e-12
        assert orthonormality_defect(f.u) <= 1e-10
        assert orthonormality_defect(f.vt.T) <= 1e-10
        lead = np.argmax(np.abs(f.u), axis=0)
        assert np.all(f.u[lead, np.arange(f.u.shape[1])] >= 0.0)
        np.testing.assert_allclose(f.u, fo.u, atol=1e-10)  # same canonical signs

    def test_known_answers(self):
        f = full_svd([[3.0, 0.0], [0.0, 0.0], [4.0, 0.0]])
        assert abs(f.s[0] - 5.0) < 1e-12 and f.s[1] == 0.0
        f = full_svd(np.eye(3))
        assert np.allclose(f.s, [1, 1, 1], atol=1e-12)
        f = full_svd(np.diag([5.0, 1e-20]))
        assert f.s[0] == 5.0 and f.s[1] == 0.0

    def test_rank_deficient(self):
        rng = np.random.default_rng(0)
        a = rng.standard_normal((10, 3)) @ rng.standard_normal((3, 7))
        f = truncated_svd(a, 3)
        assert frobenius_norm(a - reconstruct(f)) <= 1e-8
        g = full_svd(a)
        assert np.all(g.s[3:] == 0.0)
        assert orthonormality_defect(g.u) <= 1e-12

    def test_gram_eigenvalues(self):
        rng = np.random.default_rng(42)
        a = rng.standard_normal((8, 6))
        eig = np.linalg.eigvalsh(a.T @ a)[::-1]
        assert np.allclose(full_svd(a).s, np.sqrt(np.maximum(eig, 0.0)), atol=1e-8)

    def test_width_includes_exact_zeros(self):
        f = truncated_svd(np.diag([5.0, 0.0]), 2)
        assert f.s.shape == (2,) and f.s[1] == 0.0
        assert orthonormality_defect(f.u) <= 1e-12

    def test_oversized_k_caps(self):
        assert truncated_svd(np.ones((3, 2)), 10).s.shape == (2,)

    def test_rejects(self):
        with pytest.raises(ValueError):
            full_svd([[1.0, float("nan")], [0.0, 1.0]])
        with pytest.raises(ValueError):
            truncated_svd(np.eye(2), 0)

    @pytest.mark.parametrize("k", [1, 2, 4])
    def test_eckart_young(self, k):
        rng = np.random.default_rng(17)
        a = rng.standard_normal((9, 7))
        err = frobenius_norm(a - reconstruct(truncated_svd(a, k)))
        for _ in range(20):
            b = rng.standard_normal((9, k)) @ rng.standard_normal((k, 7))
            assert err <= frobenius_norm(a - b) + 1e-9


class TestMetrics:
    def test_frob_error_zero_for_full_rank(self):
        rng = np.random.default_rng(0)
        assert frob_error(SvdEngine(rng.standard_normal((6, 4)), k=4)) <= 1e-9

    def test_frob_error_equals_discarded_value(self):
        assert abs(frob_error(SvdEngine(np.diag([4.0, 3.0, 1.0]), k=2)) - 1.0) < 1e-12

    def test_frob_error_matches_host(self):
        rng = np.random.default_rng(3)
        eng = SvdEngine(rng.standard_normal((70, 50)), k=7)
        for _ in range(30):
            eng.rank_one_update(int(rng.integers(70)), int(rng.integers(50)), 0.2)
        host = frobenius_norm(eng.tracked - reconstruct(eng.factors))
        assert abs(frob_error(eng) - host) <= 1e-12 * host

    def test_never_beats_oracle(self):
        rng = np.random.default_rng(1)
        eng = SvdEngine(rng.standard_normal((15, 12)), k=4)
        for _ in range(100):
            eng.rank_one_update(int(rng.integers(15)), int(rng.integers(12)), float(rng.normal(0, 0.1)))
        assert frob_error(eng) >= compute_oracle(eng, 4).frob_opt - 1e-9
        assert frob_error(eng) >= compute_oracle(eng.tracked, 4).frob_opt - 1e-9

    def test_oracle_known_answers(self):
        frob_opt, basis, t = oracle_baseline(np.diag([4.0, 3.0]), 1)
        assert abs(frob_opt - 3.0) < 1e-12 and basis.shape == (2, 1) and t >= 0.0
        rng = np.random.default_rng(2)
        a = rng.standard_normal((9, 3)) @ rng.standard_normal((3, 8))
        assert oracle_baseline(a, 3)[0] <= 1e-9
        a = rng.standard_normal((20, 15))
        s = np.linalg.svd(a, compute_uv=False)
        assert abs(oracle_baseline(a, 4)[0] - math.sqrt(float(np.sum(s[4:] ** 2)))) <= 1e-9
        o = compute_oracle(rng.standard_normal((10, 6)), 2)
        assert o.singular_values.shape == (6,) and o.basis.shape == (10, 2)

    def test_oracle_after_refresh_reuses_the_refresh_svd(self):
        """The observation that follows an init / refresh of the same tracked
        matrix is served from that dense SVD (engine.cu: svdc_*): it must
        equal a fresh factorisation of the tracked matrix bit for bit, and any
        event must invalidate it (metrics.py:56-64, stream.py:291-333)."""
        rng = np.random.default_rng(7)
        a0 = rng.standard_normal((60, 9)) @ rng.standard_normal((9, 40)) + 0.01 * rng.standard_normal((60, 40))
        eng = SvdEngine(a0, k=6)
        for phase in range(3):
            if phase == 1:
                for _ in range(5):
                    eng.row_append(rng.standard_normal(40))
                eng.refresh()
            cached = compute_oracle(eng, 6)           # right after init / refresh
            host = compute_oracle(eng.tracked, 6)     # the same matrix through the functional entry
            np.testing.assert_allclose(cached.singular_values, host.singular_values, rtol=1e-12, atol=1e-13)
            np.testing.assert_allclose(cached.basis, host.basis, atol=1e-10)
            eng.set_rank(6)                           # same rank: only drops the cached spectrum
            fresh = compute_oracle(eng, 6)            # the resident matrix, factored again
            assert np.array_equal(cached.singular_values, fresh.singular_values)
            assert np.array_equal(cached.basis, fresh.basis)
            assert cached.frob_opt == fresh.frob_opt
            if phase == 2:
                break
            # an event invalidates: the next observation factors the new matrix
            eng.rank_one_update(3, 4, 0.5)
            after = compute_oracle(eng, 6)
            fresh = compute_oracle(eng.tracked, 6)
            assert np.array_equal(after.singular_values, fresh.singular_values)
            assert not np.array_equal(after.singular_values, cached.singular_values)
        # a different width is not served from the cache
        eng.refresh()
        assert compute_oracle(eng, 3).basis.shape == (eng.shape[0], 3)
        np.testing.assert_array_equal(compute_oracle(eng, 3).singular_values,
                                      compute_oracle(eng.tracked, 3).singular_values)

    def test_refresh_after_oracle_reuses_the_observed_svd(self):
        """The policies observe (oracle) and then refresh the same tracked
        matrix (stream.py:291-333); the refresh installs the observed leading
        triplets instead of factoring A again (engine.cu: OracleKeep).  Same
        factors as a refresh without the observation, also at a smaller armed
        rank, and an event in between drops the kept factorisation."""
        rng = np.random.default_rng(11)
        a0 = rng.standard_normal((80, 12)) @ rng.standard_normal((12, 30)) + 0.02 * rng.standard_normal((80, 30))
        rows = [rng.standard_normal(30) for _ in range(6)]

        def fresh(k_new, extra=False):
            e = SvdEngine(a0, k=8)
            for r in rows:
                e.row_append(r)
            if extra:
                e.rank_one_update(5, 7, 0.3)
            e.set_rank(k_new)
            e.refresh()
            return e.factors

        for k_new in (8, 5):
            e = SvdEngine(a0, k=8)
            for r in rows:
                e.row_append(r)
            o = compute_oracle(e, 8)
            e.set_rank(k_new)       # the armed rank of the adaptive policy
            e.refresh()
            f, g = e.factors, fresh(k_new)
            np.testing.assert_allclose(f.s, g.s, rtol=1e-13)
            np.testing.assert_allclose(f.u, g.u, atol=1e-11)
            np.testing.assert_allclose(f.vt, g.vt, atol=1e-11)
            np.testing.assert_allclose(f.s, o.singular_values[:k_new], rtol=1e-13)
            assert abs(frob_error(e) - math.sqrt(float(np.sum(o.singular_values[k_new:] ** 2)))) <= 1e-9
        e = SvdEngine(a0, k=8)
        for r in rows:
            e.row_append(r)
        compute_oracle(e, 8)
        e.rank_one_update(5, 7, 0.3)   # the tracked matrix changed: factor again
        e.refresh()
        g = fresh(8, extra=True)
        np.testing.assert_allclose(e.factors.s, g.s, rtol=1e-13)
        np.testing.assert_allclose(e.factors.u, g.u, atol=1e-11)
        # a larger rank than observed is factored again
        e = SvdEngine(a0, k=4)
        compute_oracle(e, 4)
        e.set_rank(7)
        e.refresh()
        assert e.factors.s.shape == (7,)
        np.testing.assert_allclose(e.factors.s, np.linalg.svd(a0, compute_uv=False)[:7], rtol=1e-10)

    def test_error_ratio(self):
        assert error_ratio(2.0, 2.0) == 1.0
        assert math.isnan(error_ratio(0.5, 0.0))
        assert math.isnan(error_ratio(1.0, 1e-14))

    def test_evr(self):
        rng = np.random.default_rng(5)
        assert abs(evr(SvdEngine(rng.standard_normal((6, 5)), k=5)) - 1.0) <= 1e-9
        assert abs(evr(SvdEngine(np.diag([4.0, 3.0]), k=1)) - 0.64) < 1e-12
        with pytest.raises(ValueError):
            evr(SvdEngine(np.zeros((2, 2)), k=1))

    def test_evr_full_spectrum(self):
        rng = np.random.default_rng(6)
        eng = SvdEngine(rng.standard_normal((12, 10)), k=3)
        for _ in range(50):
            eng.rank_one_update(int(rng.integers(12)), int(rng.integers(10)), float(rng.normal(0, 0.1)))
        s = np.linalg.svd(eng.tracked, compute_uv=False)
        assert abs(evr(eng) - float(np.sum(eng.factors.s ** 2)) / float(np.sum(s ** 2))) <= 1e-8

    def test_angles(self):
        eng = SvdEngine(np.eye(3), k=2)
        assert angle_to_ref(eng) is None
        eng = SvdEngine(np.eye(4), k=2)
        eng.ref_subspace = np.eye(4)[:, :2]
        u = np.zeros((4, 2)); u[2, 0] = 1.0; u[3, 1] = 1.0
        f = eng.factors
        f.u = u
        eng.factors = f
        assert abs(angle_to_ref(eng) - math.pi / 2) < 1e-12
        rng = np.random.default_rng(7)
        eng = SvdEngine(rng.standard_normal((6, 5)), k=3)
        eng.set_reference()
        eng.set_rank(2)
        assert angle_to_ref(eng) is None
        rng = np.random.default_rng(8)
        a = rng.standard_normal((10, 4)) @ rng.standard_normal((4, 8)) + 0.01 * rng.standard_normal((10, 8))
        eng = SvdEngine(a, k=4)
        assert angle_to_opt(eng, compute_oracle(eng, 4).basis) <= 1e-7

    def test_collect(self):
        eng = SvdEngine(np.diag([2.0, 1.0]), k=2)
        rec = collect(eng, update_time=0.5, refreshed=False)
        assert rec.step == 0 and rec.frob_opt is None and rec.angle_opt is None
        eng = SvdEngine(np.diag([4.0, 3.0, 1.0]), k=2)
        rec = collect(eng, 0.0, True, compute_oracle(eng, 2))
        assert abs(rec.frob_error - 1.0) < 1e-12 and abs(rec.frob_opt - 1.0) < 1e-12
        assert abs(rec.frob_ratio - 1.0) <= 1e-9 and rec.angle_opt <= 1e-8

    def test_is_defined(self):
        assert is_defined(0.0) and not is_defined(None) and not is_defined(float("nan"))


def _spec_events(m, n, k, scenario, events, seed, delta_sd=0.05):
    rng = np.random.default_rng(seed)
    a0 = rng.standard_normal((m, 3)) @ rng.standard_normal((3, n)) + 0.05 * rng.standard_normal((m, n))
    ev = []
    if scenario == "rank1":
        from paper_2605_24514_b200.stream import RankOneUpdate
        for _ in range(events):
            ev.append(RankOneUpdate(int(rng.integers(m)), int(rng.integers(n)),
                                    float(rng.normal(0, delta_sd))))
    else:
        from paper_2605_24514_b200.stream import RowAppend
        d = rng.standard_normal((6, n))
        for _ in range(events):
            ev.append(RowAppend(rng.standard_normal(6) @ d))
    return a0, ev


class TestStream:
    def test_one_record_per_event_and_cadence(self):
        a0, ev = _spec_events(20, 15, 3, "rank1", 120, 0)
        recs = run_stream(a0, ev, 3, log_every=50)
        assert [r.step for r in recs] == list(range(121))
        for r in recs:
            assert (r.frob_opt is not None) == (r.step % 50 == 0)

    def test_deterministic(self):
        a0, ev = _spec_events(20, 15, 3, "rank1", 150, 1)
        pol = PolicyConfig(kind="periodic", period=50)
        a = run_stream(a0, ev, 3, pol, log_every=50)
        b = run_stream(a0, ev, 3, pol, log_every=50)
        for ra, rb in zip(a, b):
            assert ra.frob_error == rb.frob_error and ra.evr == rb.evr
            assert ra.frob_opt == rb.frob_opt and ra.angle_opt == rb.angle_opt

    def test_periodic_refresh_flags(self):
        a0, ev = _spec_events(20, 15, 3, "rank1", 300, 2)
        recs = run_stream(a0, ev, 3, PolicyConfig(kind="periodic", period=100), log_every=100)
        assert [r.step for r in recs if r.refreshed] == [100, 200, 300]
        for r in recs:
            if r.refreshed and r.frob_ratio is not None:
                assert r.frob_ratio <= 1.0 + 1e-9

    def test_error_policy(self):
        a0, ev = _spec_events(20, 15, 3, "rank1", 600, 3, delta_sd=0.1)
        recs = run_stream(a0, ev, 3, PolicyConfig(kind="error", gamma=1.02, min_spacing=50),
                          log_every=25)
        steps = [r.step for r in recs if r.refreshed]
        assert steps and all(s % 25 == 0 for s in steps)
        assert np.all(np.diff([0] + steps) >= 50)

    def test_angle_policy(self):
        a0, ev = _spec_events(20, 15, 3, "rank1", 600, 4, delta_sd=0.1)
        recs = run_stream(a0, ev, 3, PolicyConfig(kind="angle", theta_max=0.03), log_every=25)
        steps = [r.step for r in recs if r.refreshed]
        assert steps and all(s % 25 == 0 for s in steps)

    def test_novelty_bump(self):
        a0, ev = _spec_events(20, 15, 3, "rows", 40, 5)
        pol = PolicyConfig(kind="periodic", period=20,
                           adaptive=AdaptiveRankConfig(tau=0.99, k_min=2, k_max=6, eta=0.3))
        recs, eng = run_stream(a0, ev, 3, pol, log_every=10, return_engine=True)
        assert eng.work_rank > 3 and max(r.rank for r in recs) > 3
        assert eng.shape == (60, 15)

    # ported from the reference's tests/test_stream.py simulation tests
    def test_empty_stream_single_init_record(self):
        a0, _ = _spec_events(20, 15, 3, "rank1", 0, 6)
        recs = run_stream(a0, [], 3, log_every=50)
        assert len(recs) == 1 and recs[0].step == 0
        assert is_defined(recs[0].frob_opt)

    def test_oracle_only_at_cadence(self):
        a0, ev = _spec_events(20, 15, 3, "rank1", 120, 7)
        recs = run_stream(a0, ev, 3, log_every=50)
        for r in recs:
            assert (r.opt_time is not None) == (r.step % 50 == 0)

    def test_update_time_excludes_oracle_cost(self):
        a0, ev = _spec_events(20, 15, 3, "rank1", 60, 8)
        recs = run_stream(a0, ev, 3, log_every=60)
        logged = [r for r in recs if r.step == 60][0]
        assert logged.update_time >= 0.0 and logged.opt_time >= 0.0

    def test_evr_rule_shrinks_oversized_rank(self):
        rng = np.random.default_rng(9)
        a0 = rng.standard_normal((20, 2)) @ rng.standard_normal((2, 15))
        from paper_2605_24514_b200.stream import RankOneUpdate
        ev = [RankOneUpdate(int(rng.integers(20)), int(rng.integers(15)),
                            float(rng.normal(0, 0.01))) for _ in range(120)]
        pol = PolicyConfig(kind="periodic", period=60,
                           adaptive=AdaptiveRankConfig(tau=0.999, k_min=1, k_max=8, eta=0.5))
        recs, eng = run_stream(a0, ev, 6, pol, log_every=20, return_engine=True)
        assert eng.work_rank < 6

    def test_rank1_stream_preserves_shape(self):
        a0, ev = _spec_events(20, 15, 3, "rank1", 50, 10)
        _, eng = run_stream(a0, ev, 3, log_every=50, return_engine=True)
        assert eng.shape == (20, 15)

    def test_structural_row_stream_grows_matrix(self):
        a0, ev = _spec_events(20, 15, 3, "rows", 30, 11)
        _, eng = run_stream(a0, ev, 3, log_every=50, return_engine=True)
        assert eng.shape == (50, 15)
