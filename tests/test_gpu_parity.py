"""Parity of the CUDA path against the reference: golden trajectories (made
by the real reference), the CPU oracle on seeded BASELINE-shaped inputs, and
size-independent properties at the full BASELINE sizes.

Tolerances (BASELINE.json north_star): singular values 1e-9 relative;
subspace principal angles < 1e-6 rad (sine-based, SURVEY.md 7 hard part 4);
metric trajectories (error ratio, EVR) 1e-8 relative."""

import ctypes as C

import numpy as np
import pytest

from conftest import check_sim, rel_err, sim_array, sim_inputs, sine_angle
from oracle import OracleEngine, kernel_rank_one, kernel_row_append, core_svd_jacobi
from paper_2605_24514_b200 import BatchedSvdEngine, SvdEngine, _lib, workloads
from paper_2605_24514_b200.metrics import (angle_to_opt, collect, compute_oracle, error_ratio,
                                           frob_error)

pytestmark = pytest.mark.gpu

SIGMA_RTOL = 1e-9
ANGLE_TOL = 1e-6
TRAJ_RTOL = 1e-8


# ------------------------------------------------------- functional kernels
@pytest.mark.parametrize("s", [1, 2, 5, 9, 16, 33, 64, 65, 129])
def test_core_svd_contract(s):
    import torch

    rng = np.random.default_rng(s)
    cores = rng.standard_normal((3, s, s))
    cores[2, -1, :] = 0.0  # a dead direction (_kernels.pyx:62-79 completion)
    d = torch.tensor(cores, device="cuda")
    u, vt = torch.empty_like(d), torch.empty_like(d)
    sv = torch.empty((3, s), dtype=torch.float64, device="cuda")
    lib = _lib.load()
    _lib.check(lib.isvd_core_svd(3, s, d.data_ptr(), u.data_ptr(), sv.data_ptr(), vt.data_ptr(),
                                 None))
    torch.cuda.synchronize()
    u, sv, vt = u.cpu().numpy(), sv.cpu().numpy(), vt.cpu().numpy()
    for b in range(3):
        ref = np.linalg.svd(cores[b], compute_uv=False)
        np.testing.assert_allclose((u[b] * sv[b]) @ vt[b], cores[b], atol=1e-12 * max(1, s))
        assert np.all(np.diff(sv[b]) <= 0)
        assert np.linalg.norm(u[b].T @ u[b] - np.eye(s)) <= 1e-12 * max(1, s)
        assert np.linalg.norm(vt[b] @ vt[b].T - np.eye(s)) <= 1e-12 * max(1, s)
        live = ref > 1e-12 * ref[0]
        assert rel_err(sv[b][live], ref[live]) < 1e-10
    assert sv[2][-1] == 0.0


def _functional_row_append(u, s, vt, x, tol, keep):
    lib = _lib.load()
    m, r = u.shape
    n = vt.shape[1]
    uo, so, vto = np.empty((m + 1, keep)), np.empty(keep), np.empty((keep, n))
    rho = C.c_double()
    _lib.check(lib.isvd_row_append(m, r, n, _lib.dptr(np.ascontiguousarray(u)), _lib.dptr(s),
                                   _lib.dptr(np.ascontiguousarray(vt)), _lib.dptr(x), tol, keep,
                                   _lib.dptr(uo), _lib.dptr(so), _lib.dptr(vto), C.byref(rho)))
    return uo, so, vto, rho.value


def _functional_rank_one(u, s, vt, i, j, d, keep):
    lib = _lib.load()
    m, r = u.shape
    n = vt.shape[1]
    uo, so, vto = np.empty((m, keep)), np.empty(keep), np.empty((keep, n))
    _lib.check(lib.isvd_rank_one(m, r, n, _lib.dptr(np.ascontiguousarray(u)), _lib.dptr(s),
                                 _lib.dptr(np.ascontiguousarray(vt)), i, j, d, keep, _lib.dptr(uo),
                                 _lib.dptr(so), _lib.dptr(vto)))
    return uo, so, vto


def test_functional_kernels_match_reference_golden(golden):
    u, s, vt, x = (golden[k] for k in ("ra_in_u", "ra_in_s", "ra_in_vt", "ra_in_x"))
    u2, s2, vt2, rho = _functional_row_append(u, s, vt, x, 1e-10, 5)
    for flavour in ("compiled", "python"):
        np.testing.assert_allclose(s2, golden[f"ra_{flavour}_s"], rtol=SIGMA_RTOL)
        np.testing.assert_allclose((u2 * s2) @ vt2, golden[f"ra_{flavour}_recon"], atol=1e-11)
        assert abs(rho - float(golden[f"ra_{flavour}_rho"])) <= 1e-12
    u3, s3, vt3 = _functional_rank_one(u, s, vt, 3, 6, 0.25, 4)
    for flavour in ("compiled", "python"):
        np.testing.assert_allclose(s3, golden[f"r1_{flavour}_s"], rtol=SIGMA_RTOL)
        np.testing.assert_allclose((u3 * s3) @ vt3, golden[f"r1_{flavour}_recon"], atol=1e-11)


def test_functional_row_append_contracts():
    rng = np.random.default_rng(1)
    a = rng.standard_normal((6, 5))
    f = np.linalg.svd(a, full_matrices=False)
    x = rng.standard_normal(5)
    u, s, vt, rho = _functional_row_append(f[0], f[1], f[2], x, 1e-10, 5)
    stacked = np.vstack([a, x[None, :]])
    assert rho > 0.0
    assert np.allclose((u * s) @ vt, stacked, atol=1e-9)
    # in-span row -> rho <= tol branch, exactly one zero sigma
    g = np.random.default_rng(4)
    b = g.standard_normal((7, 3)) @ g.standard_normal((3, 6))
    uu, ss, vv = np.linalg.svd(b, full_matrices=False)
    uu, ss, vv = uu[:, :3], ss[:3], vv[:3]
    x = np.array([0.4, -1.1, 0.3]) @ vv
    u2, s2, vt2, rho = _functional_row_append(uu, ss, vv, x, 1e-10, 4)
    assert rho <= 1e-10 and s2[-1] == 0.0 and np.count_nonzero(s2) == 3


def test_functional_rank_one_projection():
    rng = np.random.default_rng(2)
    b = rng.standard_normal((8, 3)) @ rng.standard_normal((3, 6))
    uu, ss, vv = np.linalg.svd(b, full_matrices=False)
    u, s, vt = uu[:, :3], ss[:3], vv[:3]
    u2, s2, vt2 = _functional_rank_one(u, s, vt, 5, 2, 0.7, 3)
    bump = np.zeros((8, 6))
    bump[5, 2] = 0.7
    proj = (u @ u.T) @ ((u * s) @ vt + bump) @ (vt.T @ vt)
    assert np.allclose((u2 * s2) @ vt2, proj, atol=1e-10)


@pytest.mark.parametrize("keep", [3, 4])
def test_functional_matches_oracle_kernels(keep):
    rng = np.random.default_rng(keep)
    b = rng.standard_normal((50, 3)) @ rng.standard_normal((3, 40)) + 0.1 * rng.standard_normal((50, 40))
    uu, ss, vv = np.linalg.svd(b, full_matrices=False)
    u, s, vt = uu[:, :3].copy(), ss[:3].copy(), vv[:3].copy()
    x = rng.standard_normal(40)
    g = _functional_row_append(u, s, vt, x, 1e-10, keep)
    o = kernel_row_append(u, s, vt, x, 1e-10, keep, core_svd_jacobi)
    assert rel_err(g[1], o[1]) < SIGMA_RTOL
    np.testing.assert_allclose((g[0] * g[1]) @ g[2], (o[0] * o[1]) @ o[2], atol=1e-11)


# ------------------------------------------------------- golden trajectories
def _run_traj(a0, events, k, kind=None, period=None, gamma=None, theta=None):
    eng = SvdEngine(a0, k)
    eng.set_reference()
    recs = []
    for t, ev in enumerate(events, start=1):
        if ev[0] == "row":
            eng.row_append(ev[1])
        elif ev[0] == "col":
            eng.col_append(ev[1])
        else:
            eng.rank_one_update(ev[1], ev[2], ev[3])
        orc = compute_oracle(eng, eng.work_rank)
        fire = False
        if kind == "periodic":
            fire = t % period == 0
        elif kind == "error":
            r = error_ratio(frob_error(eng), orc.frob_opt)
            fire = (not np.isnan(r)) and r > gamma
        elif kind == "angle":
            fire = angle_to_opt(eng, orc.basis) > theta
        if fire:
            eng.refresh(store_reference=True)
        rec = collect(eng, 0.0, fire, orc)
        recs.append([rec.frob_error, rec.evr, rec.rank, float(rec.refreshed), rec.frob_opt,
                     rec.frob_ratio if rec.frob_ratio is not None else np.nan, rec.angle_opt])
    return np.array(recs), eng


def _check(golden, tag, recs, eng):
    ref = golden[f"traj_{tag}_records"]
    np.testing.assert_array_equal(recs[:, 2:4], ref[:, 2:4])
    np.testing.assert_allclose(recs[:, [0, 1, 4]], ref[:, [0, 1, 4]], rtol=TRAJ_RTOL, atol=1e-12)
    ok = ~np.isnan(ref[:, 5])
    np.testing.assert_array_equal(np.isnan(recs[:, 5]), ~ok)
    np.testing.assert_allclose(recs[ok, 5], ref[ok, 5], rtol=TRAJ_RTOL)
    assert np.max(np.abs(recs[:, 6] - ref[:, 6])) < ANGLE_TOL  # angle_opt
    f = eng.factors
    np.testing.assert_allclose(f.s, golden[f"traj_{tag}_s"], rtol=SIGMA_RTOL)
    assert sine_angle(f.u, golden[f"traj_{tag}_u"]) < ANGLE_TOL
    assert sine_angle(f.vt.T, golden[f"traj_{tag}_vt"].T) < ANGLE_TOL
    np.testing.assert_allclose(f.u, golden[f"traj_{tag}_u"], atol=1e-7)  # canonical signs
    assert abs(eng.sq_norm - float(golden[f"traj_{tag}_sq_norm"])) <= 1e-12 * eng.sq_norm


# whole BASELINE streams through the product loop (stream.run_stream) vs the
# reference's own run_simulation on the same inputs (make_golden.py): cfg1
# (1000 appends), cfg2 (2000 rank-1 updates, error trigger), cfg3 (all 2268
# daily appends, angle trigger), config 4 at reduced size with the adaptive
# rank policy (EVR selection, hysteresis, armed rank at refresh; and a
# variant where the novelty bump fires), and the reortho guard forced on
# every tick.
@pytest.mark.parametrize("tag", ["cfg1", "cfg2", "cfg3", "cfg4r", "cfg4b", "guard"])
def test_reference_loop_trajectory(golden, tag, monkeypatch):
    import paper_2605_24514_b200.engine as E
    from paper_2605_24514_b200.policies import AdaptiveRankConfig, PolicyConfig
    from paper_2605_24514_b200.stream import run_stream

    a0, ev, k, pol, log_every = sim_inputs(golden, tag)
    guard = tag == "guard"
    if guard:  # as the reference's tests/test_engine.py:309-311
        monkeypatch.setattr(E, "REORTHO_THRESHOLD", -1.0)
    ad = pol.pop("adaptive", None)
    policy = PolicyConfig(**pol, adaptive=AdaptiveRankConfig(**ad) if ad else None)
    recs, eng = run_stream(a0, workloads.to_stream_events(ev), k, policy, log_every,
                           reortho_guard=guard, return_engine=True)
    check_sim(golden, tag, sim_array(recs))
    f = eng.factors
    np.testing.assert_allclose(f.s, golden[f"sim_{tag}_s"], rtol=SIGMA_RTOL)
    assert sine_angle(f.u, golden[f"sim_{tag}_u"]) < ANGLE_TOL
    assert sine_angle(f.vt.T, golden[f"sim_{tag}_vt"].T) < ANGLE_TOL
    np.testing.assert_allclose(f.u, golden[f"sim_{tag}_u"], atol=1e-7)  # canonical signs
    assert abs(eng.sq_norm - float(golden[f"sim_{tag}_sq_norm"])) <= 1e-12 * eng.sq_norm


def test_golden_mixed(golden):
    from test_oracle_golden import _mixed_events

    recs, eng = _run_traj(golden["traj_mixed_a0"], _mixed_events(golden), 6)
    _check(golden, "mixed", recs, eng)


# ------------------------------------------------------------- batched 5a
def _oracle_stream(a0, events, k):
    oe = OracleEngine(a0, k)
    for e in events:
        if e[0] == "row":
            oe.row_append(e[1])
        else:
            oe.rank_one_update(e[1], e[2], e[3])
    return oe


def _run_batched(eng, ticks):
    for tk in ticks:
        if tk[0] == "row":
            eng.row_append(tk[1])
        else:
            eng.rank_one_update(tk[1], tk[2], tk[3])


@pytest.mark.parametrize("n,k,B", [(7, 3, 1), (33, 8, 1), (100, 12, 1), (255, 20, 1), (256, 24, 1),
                                    (64, 31, 1), (50, 5, 70), (200, 17, 70), (256, 32, 66)])
def test_row_append_projection_shapes(n, k, B):
    """The narrow-stream projection kernel (project_append32_kernel<LD>, every
    factor pitch 8 / 16 / 24 / 32; B >= 64 turns the deferred right basis on:
    appended residuals Z and the small G) over ragged widths, mixed with
    rank-1 updates so G is not the identity: factors, tracked matrix and N
    against the oracle engine of each stream (_kernels.pyx:135-157)."""
    rng = np.random.default_rng(1000 * n + k)
    m0, T = max(k + 3, 24), 21
    x0 = rng.standard_normal((B, m0, min(k, n))) @ rng.standard_normal((B, min(k, n), n))
    a0 = x0 + 0.05 * rng.standard_normal((B, m0, n))
    eng = BatchedSvdEngine(a0, k, m_cap=m0 + T)
    streams = [[] for _ in range(B)]
    for t in range(T):
        if t % 3 == 2:
            i = rng.integers(0, eng.shape[0], B)
            j = rng.integers(0, n, B)
            d = 0.1 * rng.standard_normal(B)
            eng.rank_one_update(i, j, d)
            for b in range(B):
                streams[b].append(("r1", int(i[b]), int(j[b]), float(d[b])))
        else:
            rows = rng.standard_normal((B, n))
            if t == 7:
                rows[0] = 0.0  # a zero row: rho <= tol branch
            eng.row_append(rows)
            for b in range(B):
                streams[b].append(("row", rows[b].copy()))
    sq, _, _ = eng.scalars()
    for b in sorted({0, B // 2, B - 1}):
        oe = _oracle_stream(a0[b], streams[b], k)
        f = eng.factors(b)
        assert rel_err(f.s, oe.factors.s) < SIGMA_RTOL, (b, f.s, oe.factors.s)
        live = oe.factors.s > 1e-9 * oe.factors.s[0]
        assert sine_angle(f.u[:, live], oe.factors.u[:, live]) < ANGLE_TOL, b
        assert sine_angle(f.vt.T[:, live], oe.factors.vt.T[:, live]) < ANGLE_TOL, b
        assert np.array_equal(eng.tracked(b), oe.tracked), b
        assert abs(sq[b] - oe.sq_norm) <= 1e-12 * oe.sq_norm, b


@pytest.mark.parametrize("n,k", [(130, 128), (520, 40), (1000, 100), (1024, 128), (700, 130)])
def test_wide_single_stream_row_appends(n, k):
    """Few streams with wide factors (config 5b's shape class): the cluster
    projection (register-resident slices of <= 64 rows per CTA for k <= 128,
    the general cluster kernel above), the 16-CTA / 8-CTA cluster secular
    solver and the column-split rotation, against the oracle engine."""
    rng = np.random.default_rng(n + k)
    m0 = k + 12
    a0 = rng.standard_normal((m0, k)) @ rng.standard_normal((k, n)) + 1e-3 * rng.standard_normal((m0, n))
    eng, oe = SvdEngine(a0, k), OracleEngine(a0, k)
    for t in range(7):
        if t == 3:
            i, j, d = int(rng.integers(m0)), int(rng.integers(n)), float(rng.normal(0, 0.1))
            eng.rank_one_update(i, j, d)
            oe.rank_one_update(i, j, d)
        else:
            x = rng.standard_normal(k) @ a0[:k] + 1e-3 * rng.standard_normal(n)
            eng.row_append(x)
            oe.row_append(x)
    f, g = eng.factors, oe.factors
    assert rel_err(f.s, g.s) < SIGMA_RTOL
    live = g.s > 1e-6 * g.s[0]
    assert sine_angle(f.u[:, live], g.u[:, live]) < ANGLE_TOL
    assert sine_angle(f.vt.T[:, live], g.vt.T[:, live]) < ANGLE_TOL
    assert np.array_equal(eng.tracked, oe.tracked)
    assert abs(eng.sq_norm - oe.sq_norm) <= 1e-12 * oe.sq_norm


def test_cfg5a_batched_matches_oracle():
    """8 streams, 64 interleaved events each, through the batched engine vs
    one oracle engine per stream."""
    B, T = 8, 64
    a0, ticks, streams = workloads.cfg5a_batch(0, B, n_events=T)
    eng = BatchedSvdEngine(a0, 32, m_cap=1024 + T)
    _run_batched(eng, ticks)
    for b in range(B):
        oe = _oracle_stream(*streams[b], 32)
        f = eng.factors(b)
        assert rel_err(f.s, oe.factors.s) < SIGMA_RTOL
        assert sine_angle(f.u, oe.factors.u) < ANGLE_TOL
        assert sine_angle(f.vt.T, oe.factors.vt.T) < ANGLE_TOL
        assert np.array_equal(eng.tracked(b), oe.tracked)
    sq, rho, xn = eng.scalars()
    for b in range(B):
        assert abs(sq[b] - float(np.sum(eng.tracked(b) ** 2))) <= 1e-12 * sq[b]


def test_cfg5a_benchmarked_configuration(golden):
    """The exact path bench.py times: config 5a shape (1024 x 256, rank 32,
    k = 32, all 1024 alternating events) on a 512-stream batch, so the
    deferred right basis (B >= 64) and the four run-ahead stream groups
    (B >= 512) are on, with the default deferred-U window.  Eight sampled
    streams are replayed through the oracle (sigma 1e-9, sine angles 1e-6,
    tracked matrix and N bit-exact / 1e-12); streams 0 and 1 also against the
    reference's own 1024-event output."""
    B, T = 512, 1024
    a0, ticks, streams = workloads.cfg5a_batch(0, B, n_events=T)
    eng = BatchedSvdEngine(a0, 32, m_cap=1024 + T // 2 + 1, k_cap=32)
    del a0
    _run_batched(eng, ticks)
    eng.flush()
    assert eng.shape == (1536, 256)
    sq, _, _ = eng.scalars()
    for b in (0, 1, 63, 64, 127, 255, 256, 383, 384, 511):
        oe = _oracle_stream(*streams[b], 32)
        f = eng.factors(b)
        assert rel_err(f.s, oe.factors.s) < SIGMA_RTOL, b
        assert sine_angle(f.u, oe.factors.u) < ANGLE_TOL, b
        assert sine_angle(f.vt.T, oe.factors.vt.T) < ANGLE_TOL, b
        np.testing.assert_allclose(f.u, oe.factors.u, atol=1e-8)  # canonical signs
        assert np.array_equal(eng.tracked(b), oe.tracked), b
        assert abs(sq[b] - oe.sq_norm) <= 1e-12 * oe.sq_norm, b
        if b < 2:
            assert rel_err(f.s, golden[f"s5a_{b}_s"]) < SIGMA_RTOL
            assert sine_angle(f.vt.T, golden[f"s5a_{b}_vt"].T) < ANGLE_TOL
            np.testing.assert_allclose(f.u[:64], golden[f"s5a_{b}_u"], atol=1e-8)
    du, dv = eng.ortho_defect()
    assert np.all(du <= 1e-10) and np.all(dv <= 1e-10)


def test_cfg5a_full_length_properties():
    """Full 1024-event streams (BASELINE config 5a shape) on a 16-stream
    batch: size-independent properties (orthonormality, N_t identity,
    optimality of the truncation error) plus oracle parity on two streams."""
    B, T = 16, 1024
    a0, ticks, streams = workloads.cfg5a_batch(1, B, n_events=T)
    eng = BatchedSvdEngine(a0, 32, m_cap=1024 + T // 2)
    for tk in ticks:
        if tk[0] == "row":
            eng.row_append(tk[1])
        else:
            eng.rank_one_update(tk[1], tk[2], tk[3])
    assert eng.shape == (1536, 256)
    du, dv = eng.ortho_defect()
    assert np.all(du <= 1e-8) and np.all(dv <= 1e-8)
    sq, _, _ = eng.scalars()
    err = eng.frob_error()
    s_all, _ = eng.oracle(32)
    opt = np.sqrt(np.sum(s_all[:, 32:] ** 2, axis=1))
    for b in range(B):
        direct = float(np.sum(eng.tracked(b) ** 2))
        assert abs(sq[b] - direct) <= 1e-9 * direct
        assert err[b] >= opt[b] - 1e-9
        assert err[b] / opt[b] < 1.2
    for b in (0, B - 1):
        oe = OracleEngine(streams[b][0], 32)
        for e in streams[b][1]:
            if e[0] == "row":
                oe.row_append(e[1])
            else:
                oe.rank_one_update(e[1], e[2], e[3])
        f = eng.factors(b)
        assert rel_err(f.s, oe.factors.s) < SIGMA_RTOL
        assert sine_angle(f.u, oe.factors.u) < ANGLE_TOL


# ------------------------------------------- append-core solver cross-checks
def _solver(eng, jacobi: bool):
    _lib.check(eng._h.lib.isvd_engine_set_append_solver(eng._h.h, int(jacobi)))
    return eng


HARD_CASES = [
    ("identity_equal_poles", np.eye(3), 3, [np.array([1.0, 2.0, 3.0])]),
    ("zero_sigma_present", np.diag([5.0, 0.0]), 2, [np.array([0.3, -0.7])]),
    ("pythagorean", np.array([[3.0, 0.0], [0.0, 0.0]]), 2, [np.array([4.0, 0.0])]),
    ("zero_row", np.diag([3.0, 2.0, 1.0]), 3, [np.zeros(3)]),
    ("rank_deficient_many_zeros", np.outer(np.arange(1.0, 7.0), np.ones(5)), 5,
     [np.arange(5.0), np.ones(5), np.zeros(5)]),
    ("repeated_sigma_block", np.kron(np.eye(3), np.ones((2, 2))), 4,
     [np.linspace(-1, 1, 6), np.full(6, 0.5)]),
    ("tiny_and_huge", np.diag([1e8, 1.0, 1e-6, 1e-9]), 4, [np.array([1e-3, 2.0, -1e-7, 5.0])]),
]


@pytest.mark.parametrize("name, a0, k, rows", HARD_CASES, ids=[c[0] for c in HARD_CASES])
def test_append_solver_hard_cases(name, a0, k, rows):
    """Secular-equation append solver vs the generic Jacobi solver vs the
    oracle on deflation-heavy cores (equal poles, zero poles, zero z)."""
    gs = SvdEngine(a0, k)
    gj = _solver(SvdEngine(a0, k), True)
    oc = OracleEngine(a0, k)
    for x in rows:
        x = np.resize(x, gs.shape[1])
        gs.row_append(x)
        gj.row_append(x)
        oc.row_append(x)
        yc = np.linspace(0.2, -0.4, gs.shape[0])
        gs.col_append(yc)
        gj.col_append(yc)
        oc.col_append(yc)
    for g in (gs, gj):
        f = g.factors
        fo = oc.factors
        np.testing.assert_allclose(f.s, fo.s, rtol=1e-9, atol=1e-12 * fo.s[0])
        np.testing.assert_allclose((f.u * f.s) @ f.vt, (fo.u * fo.s) @ fo.vt,
                                   atol=1e-10 * max(1.0, fo.s[0]))
        du, dv = g.ortho_defects()
        assert du <= 1e-10 and dv <= 1e-10


def test_append_solvers_agree_on_streams():
    rng = np.random.default_rng(77)
    a0 = rng.standard_normal((80, 40)) @ np.diag(np.logspace(0, -3, 40)) @ rng.standard_normal((40, 40))
    gs = SvdEngine(a0, 12)
    gj = _solver(SvdEngine(a0, 12), True)
    for t in range(200):
        if t % 2:
            x = rng.standard_normal(gs.shape[1])
            gs.row_append(x); gj.row_append(x)
        else:
            y = rng.standard_normal(gs.shape[0])
            gs.col_append(y); gj.col_append(y)
    fs, fj = gs.factors, gj.factors
    assert rel_err(fs.s, fj.s) < 1e-11
    assert sine_angle(fs.u, fj.u) < 1e-9
    np.testing.assert_allclose(fs.u, fj.u, atol=1e-9)


# ------------------------------------------------ deferred (lazy) U rotation
@pytest.mark.parametrize("k", [5, 32])
def test_lazy_and_eager_rotation_agree(k):
    """The deferred left-basis rotation (U = [Ub 0; 0 I] W, flushed every 32
    appended rows) reproduces the eager per-event rotation."""
    rng = np.random.default_rng(k)
    a0 = rng.standard_normal((120, 60)) @ np.diag(np.logspace(0, -2, 60)) @ rng.standard_normal((60, 60))
    lazy, eager, cpu = SvdEngine(a0, k), SvdEngine(a0, k), OracleEngine(a0, k)
    eager.set_lazy(False)
    for t in range(150):
        kind = t % 5
        if kind in (0, 2):
            x = rng.standard_normal(lazy.shape[1])
            for e in (lazy, eager, cpu):
                e.row_append(x)
        elif kind == 4 and t % 25 == 4:
            y = rng.standard_normal(lazy.shape[0])
            for e in (lazy, eager, cpu):
                e.col_append(y)
        else:
            i, j = int(rng.integers(lazy.shape[0])), int(rng.integers(lazy.shape[1]))
            d = float(rng.normal(0, 0.2))
            for e in (lazy, eager, cpu):
                e.rank_one_update(i, j, d)
        if t % 37 == 0:  # observation mid-window flushes
            assert lazy.factors.rank == eager.factors.rank
    fl, fe, fc = lazy.factors, eager.factors, cpu.factors
    assert rel_err(fl.s, fe.s) < 1e-11
    np.testing.assert_allclose(fl.u, fe.u, atol=1e-9)
    assert rel_err(fl.s, fc.s) < SIGMA_RTOL
    assert sine_angle(fl.u, fc.u) < ANGLE_TOL
    du, dv = lazy.ortho_defects()
    assert du < 1e-10 and dv < 1e-10


def test_batched_lazy_flush_cycle():
    """Batched 5a-shaped streams across several flush windows (32 rows each)
    with rank-1 gathers hitting both base rows and rows appended inside the
    current window."""
    B, T = 4, 200
    a0, ticks, streams = workloads.cfg5a_batch(3, B, m=200, n=64, rank=8, n_events=T)
    eng = BatchedSvdEngine(a0, 8, m_cap=200 + T)
    for t, tk in enumerate(ticks):
        if tk[0] == "row":
            eng.row_append(tk[1])
        else:
            # force gathers into the freshly appended rows half of the time
            ii = tk[1].copy()
            if t % 4 == 1:
                ii[:] = eng.shape[0] - 1
                for b in range(B):
                    streams[b][1][t] = ("rank1", int(ii[b]), int(tk[2][b]), float(tk[3][b]))
            eng.rank_one_update(ii, tk[2], tk[3])
    for b in range(B):
        oe = OracleEngine(streams[b][0], 8)
        for e in streams[b][1]:
            if e[0] == "row":
                oe.row_append(e[1])
            else:
                oe.rank_one_update(e[1], e[2], e[3])
        f = eng.factors(b)
        assert rel_err(f.s, oe.factors.s) < SIGMA_RTOL
        assert sine_angle(f.u, oe.factors.u) < ANGLE_TOL
        np.testing.assert_allclose(f.u, oe.factors.u, atol=1e-8)


def test_snapshot_restore_and_groups_reproduce():
    """Batched engine with B >= 512 runs its ticks in 4 stream groups on
    separate CUDA streams; snapshot/restore replays the same ticks; both
    runs give bit-identical factors, and stream b matches the oracle."""
    B, T = 512, 24
    a0, ticks, streams = workloads.cfg5a_batch(4, B, m=96, n=48, rank=6, n_events=T)
    eng = BatchedSvdEngine(a0, 6, m_cap=96 + T)
    eng.snapshot()
    outs = []
    for rep in range(2):
        if rep:
            eng.restore()
        for tk in ticks:
            if tk[0] == "row":
                eng.row_append(tk[1])
            else:
                eng.rank_one_update(tk[1], tk[2], tk[3])
        outs.append([eng.factors(b) for b in (0, 257, B - 1)])
    for fa, fb in zip(*outs):
        assert np.array_equal(fa.s, fb.s) and np.array_equal(fa.u, fb.u)
    for idx, b in enumerate((0, 257, B - 1)):
        oe = OracleEngine(streams[b][0], 6)
        for e in streams[b][1]:
            if e[0] == "row":
                oe.row_append(e[1])
            else:
                oe.rank_one_update(e[1], e[2], e[3])
        assert rel_err(outs[0][idx].s, oe.factors.s) < SIGMA_RTOL
        assert sine_angle(outs[0][idx].u, oe.factors.u) < ANGLE_TOL


def test_benchmark_shape_ticks_are_bitwise_reproducible():
    """Config-5a-shaped ticks (1024 x 256, k = 32: the narrow-stream
    projection, the CTA-per-core kernels with their fused rotations, V
    materialisations and a U flush) replayed from a snapshot: every stream's
    factors, tracked norm and residuals must come out bit for bit the same
    (a race in any of the tick kernels shows up as a differing bit; the pool
    does not allow compute-sanitizer)."""
    B, T = 128, 100
    a0, ticks, _ = workloads.cfg5a_batch(9, B, n_events=T)
    eng = BatchedSvdEngine(a0, 32, m_cap=1024 + T // 2 + 1, k_cap=32)
    del a0
    eng.snapshot()
    outs = []
    for rep in range(2):
        if rep:
            eng.restore()
        _run_batched(eng, ticks)
        eng.flush()
        outs.append(([eng.factors(b) for b in range(0, B, 7)], [np.array(v) for v in eng.scalars()]))
    for fa, fb in zip(outs[0][0], outs[1][0]):
        assert np.array_equal(fa.s, fb.s) and np.array_equal(fa.u, fb.u) and np.array_equal(fa.vt, fb.vt)
    for va, vb in zip(outs[0][1], outs[1][1]):
        assert np.array_equal(va, vb)


def test_wide_stream_ticks_are_bitwise_reproducible():
    """The same check on a config-5b-shaped stream (1024 columns, k = 128):
    cluster projection, cluster secular solver with staged vector stores,
    column-split rotation."""
    rng = np.random.default_rng(5)
    m0, n, k, T = 4096, 1024, 128, 12
    y = rng.standard_normal((n, k))
    a0 = rng.standard_normal((m0, k)) @ y.T + 1e-3 * rng.standard_normal((m0, n))
    rows = rng.standard_normal((T, k)) @ y.T
    eng = BatchedSvdEngine(a0[None], k, m_cap=m0 + T + 1, k_cap=k)
    eng.snapshot()
    outs = []
    for rep in range(2):
        if rep:
            eng.restore()
        for t in range(T):
            eng.row_append(rows[t:t + 1])
        eng.flush()
        outs.append(eng.factors(0))
    fa, fb = outs
    assert np.array_equal(fa.s, fb.s) and np.array_equal(fa.u, fb.u) and np.array_equal(fa.vt, fb.vt)


@pytest.mark.parametrize("kappa", [99.0, 101.0, 5e3])
def test_rank_one_orthogonality_near_the_structure_gate(kappa):
    """Long rank-1 streams whose spectrum sits just inside (99) and just
    outside (101) the sigma_max / sigma_min <= 100 gate of the structured
    right-vector path, and far outside it (5e3): the factors stay orthonormal
    to the reference's level (its one-sided Jacobi stops at 1e-14,
    _kernels.pyx:38-59) over 2000 ticks, and match the oracle."""
    rng = np.random.default_rng(int(kappa))
    m, n, k, T = 160, 96, 20, 2000
    qu = np.linalg.qr(rng.standard_normal((m, k)))[0]
    qv = np.linalg.qr(rng.standard_normal((n, k)))[0]
    sig = np.geomspace(10.0, 10.0 / kappa, k)
    a0 = (qu * sig) @ qv.T
    B = 64  # batched: deferred right basis and the fused rank-1 kernel, as config 5a
    eng = BatchedSvdEngine(np.repeat(a0[None], B, axis=0), k)
    oe = OracleEngine(a0, k)
    ii, jj = rng.integers(0, m, T), rng.integers(0, n, T)
    dd = rng.normal(0.0, 1e-3, T)
    for t in range(T):
        eng.rank_one_update(np.full(B, ii[t]), np.full(B, jj[t]), np.full(B, dd[t]))
        oe.rank_one_update(int(ii[t]), int(jj[t]), float(dd[t]))
    du, dv = eng.ortho_defect()
    assert np.max(du) <= 5e-12 and np.max(dv) <= 5e-12, (np.max(du), np.max(dv))
    f = eng.factors(0)
    assert rel_err(f.s, oe.factors.s) < SIGMA_RTOL
    assert sine_angle(f.u, oe.factors.u) < ANGLE_TOL
    assert sine_angle(f.vt.T, oe.factors.vt.T) < ANGLE_TOL


def test_rank_one_fast_and_fallback_cores_in_one_launch():
    """One batched rank-1 launch holding every kind of core: streams with a
    well-separated spectrum take the structured simultaneous steps, streams
    with a repeated singular value (first-order angle above its cap) or
    sigma_max / sigma_min > 100 the in-CTA Jacobi sweeps, and delta == 0
    entries the one-warp kernel's exact path (list mode).  Every stream
    matches its own oracle, and both the step and the sweep paths ran."""
    rng = np.random.default_rng(11)
    m, n, k, T, B = 72, 48, 12, 40, 48
    a0s = []
    for b in range(B):
        qu = np.linalg.qr(rng.standard_normal((m, k)))[0]
        qv = np.linalg.qr(rng.standard_normal((n, k)))[0]
        kind = b % 3
        if kind == 0:
            sig = np.linspace(10.0, 2.0, k)            # fast path
        elif kind == 1:
            sig = np.linspace(10.0, 2.0, k)
            sig[4] = sig[3]                             # repeated value: fallback
        else:
            sig = np.geomspace(10.0, 10.0 / 500.0, k)   # outside the kappa gate: fallback
        a0s.append((qu * sig) @ qv.T)
    a0 = np.stack(a0s)
    eng = BatchedSvdEngine(a0, k)
    oes = [OracleEngine(a0[b], k) for b in range(B)]
    lib = _lib.load()
    cnt = (C.c_int64 * 8)()
    lib.isvd_debug_counters(cnt, 1)
    for t in range(T):
        ii, jj = rng.integers(0, m, B), rng.integers(0, n, B)
        dd = rng.normal(0.0, 1e-2, B)
        if t % 4 == 0:
            dd[::5] = 0.0
        eng.rank_one_update(ii, jj, dd)
        for b in range(B):
            oes[b].rank_one_update(int(ii[b]), int(jj[b]), float(dd[b]))
    eng.synchronize()
    lib.isvd_debug_counters(cnt, 1)
    cores, fast = cnt[1], cnt[7]
    assert cores == B * T and 0 < fast < cores, (cores, fast)
    du, dv = eng.ortho_defect()
    assert np.max(du) <= 1e-12 and np.max(dv) <= 1e-12
    for b in range(B):
        f, fo = eng.factors(b), oes[b].factors
        assert rel_err(f.s, fo.s) < SIGMA_RTOL, b
        assert sine_angle(f.u, fo.u) < ANGLE_TOL, b
        assert sine_angle(f.vt.T, fo.vt.T) < ANGLE_TOL, b
        assert np.array_equal(eng.tracked(b), oes[b].tracked), b


def test_row_append_cta_and_fallback_cores_in_one_launch():
    """Batched row appends (deferred bases, fused epilogue) whose cores go
    both ways in one launch: ordinary rows take the CTA-per-core secular
    kernel; in-span rows of exactly low-rank streams (rho below tol, a zero
    z entry) and zero rows need deflation and are handed to the one-warp
    kernel (list mode).  Every stream matches its own oracle."""
    rng = np.random.default_rng(12)
    B, m, n, k, T = 64, 60, 40, 12, 36
    ys = [rng.standard_normal((n, k)) for _ in range(B)]
    a0 = np.stack([rng.standard_normal((m, k)) @ ys[b].T +
                   (0.0 if b % 3 == 0 else 0.05) * rng.standard_normal((m, n)) for b in range(B)])
    eng = BatchedSvdEngine(a0, k)
    oes = [OracleEngine(a0[b], k) for b in range(B)]
    for t in range(T):
        x = np.empty((B, n))
        for b in range(B):
            if b % 3 == 0:
                x[b] = ys[b] @ rng.standard_normal(k)  # in the row space: rho ~ 0
            elif b % 3 == 1 and t % 5 == 0:
                x[b] = 0.0
            else:
                x[b] = ys[b] @ rng.standard_normal(k) + 0.05 * rng.standard_normal(n)
        eng.row_append(x)
        for b in range(B):
            oes[b].row_append(x[b])
    du, dv = eng.ortho_defect()
    assert np.max(du) <= 1e-12 and np.max(dv) <= 1e-12
    for b in range(B):
        f, fo = eng.factors(b), oes[b].factors
        assert rel_err(f.s, fo.s) < SIGMA_RTOL, b
        assert sine_angle(f.u, fo.u) < ANGLE_TOL, b
        assert sine_angle(f.vt.T, fo.vt.T) < ANGLE_TOL, b
        assert np.array_equal(eng.tracked(b), oes[b].tracked), b
