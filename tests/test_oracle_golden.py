"""Pin the CPU oracle against golden vectors produced by the real reference
(tests/golden/make_golden.py imports /root/reference and runs both of its
kernel backends).  CPU only."""

import numpy as np
import pytest

from conftest import check_sim, rel_err, sim_array, sim_inputs, sine_angle
from oracle import (AdaptiveRankConfig, OracleEngine, PolicyConfig, angle_to_opt, collect,
                    compute_oracle, core_svd_jacobi, core_svd_lapack, error_ratio, frob_error,
                    kernel_rank_one, kernel_row_append, run_stream)
from paper_2605_24514_b200 import workloads

CORES = ["rand1", "rand2", "rand5", "rand9", "rand16", "rand33", "dead", "brand33"]


@pytest.mark.parametrize("key", CORES)
@pytest.mark.parametrize("flavour", ["compiled", "python"])
def test_core_svd_matches_reference(golden, key, flavour):
    core = golden[f"core_{flavour}_{key}_in"]
    fn = core_svd_jacobi if flavour == "compiled" else core_svd_lapack
    u, s, vt = fn(core)
    np.testing.assert_allclose(s, golden[f"core_{flavour}_{key}_s"], rtol=1e-12, atol=1e-13)
    np.testing.assert_allclose((u * s) @ vt, golden[f"core_{flavour}_{key}_recon"], atol=1e-12)
    assert np.linalg.norm(u.T @ u - np.eye(len(s))) < 1e-12
    assert np.all(np.diff(s) <= 0)


@pytest.mark.parametrize("flavour", ["compiled", "python"])
def test_kernel_contracts_match_reference(golden, flavour):
    u, s, vt, x = (golden[k] for k in ("ra_in_u", "ra_in_s", "ra_in_vt", "ra_in_x"))
    fn = core_svd_jacobi if flavour == "compiled" else core_svd_lapack
    u2, s2, vt2, rho = kernel_row_append(u, s, vt, x, 1e-10, 5, fn)
    np.testing.assert_allclose(s2, golden[f"ra_{flavour}_s"], rtol=1e-12)
    np.testing.assert_allclose((u2 * s2) @ vt2, golden[f"ra_{flavour}_recon"], atol=1e-12)
    assert abs(rho - float(golden[f"ra_{flavour}_rho"])) < 1e-14
    u3, s3, vt3 = kernel_rank_one(u, s, vt, 3, 6, 0.25, 4, fn)
    np.testing.assert_allclose(s3, golden[f"r1_{flavour}_s"], rtol=1e-12)
    np.testing.assert_allclose((u3 * s3) @ vt3, golden[f"r1_{flavour}_recon"], atol=1e-12)


def _trajectory(a0, events, k, kind=None, period=None, gamma=None, theta=None):
    eng = OracleEngine(a0, k)
    eng.set_reference()
    recs = []
    for t, ev in enumerate(events, start=1):
        if ev[0] == "row":
            eng.row_append(ev[1])
        elif ev[0] == "col":
            eng.col_append(ev[1])
        else:
            eng.rank_one_update(ev[1], ev[2], ev[3])
        orc = compute_oracle(eng.tracked, eng.work_rank)
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
        rec = collect(eng, fire, orc)
        recs.append([rec.frob_error, rec.evr, rec.rank, float(rec.refreshed), rec.frob_opt,
                     rec.frob_ratio if rec.frob_ratio is not None else np.nan, rec.angle_opt])
    return np.array(recs), eng


def _check_traj(golden, tag, recs, eng):
    ref = golden[f"traj_{tag}_records"]
    assert recs.shape == ref.shape
    # columns: frob_error, evr, rank, refreshed, frob_opt, ratio, angle_opt
    np.testing.assert_array_equal(recs[:, 2:4], ref[:, 2:4])
    np.testing.assert_allclose(recs[:, [0, 1, 4]], ref[:, [0, 1, 4]], rtol=1e-8, atol=1e-12)
    ok = ~np.isnan(ref[:, 5])
    np.testing.assert_array_equal(np.isnan(recs[:, 5]), ~ok)
    np.testing.assert_allclose(recs[ok, 5], ref[ok, 5], rtol=1e-8)
    assert np.max(np.abs(recs[:, 6] - ref[:, 6])) < 1e-6
    np.testing.assert_allclose(eng.factors.s, golden[f"traj_{tag}_s"], rtol=1e-9)
    assert sine_angle(eng.factors.u, golden[f"traj_{tag}_u"]) < 1e-6
    assert abs(eng.sq_norm - float(golden[f"traj_{tag}_sq_norm"])) <= 1e-12 * eng.sq_norm


# whole-stream trajectories through the reference's own loop
# (stream.py:257-333); cfg2's oracle is a 1000 x 500 SVD per tick, so the CPU
# suite checks a prefix of it (the GPU suite runs all of it)
SIM_PREFIX = {"cfg1": None, "cfg2": 150, "cfg3": None, "cfg4r": None, "cfg4b": None,
              "guard": None}


@pytest.mark.parametrize("tag", list(SIM_PREFIX))
def test_oracle_matches_reference_loop(golden, tag, monkeypatch):
    import oracle.isvd_oracle as O

    a0, ev, k, pol, log_every = sim_inputs(golden, tag)
    n = SIM_PREFIX[tag]
    if n is not None:
        ev = ev[:n - 1]
    guard = tag == "guard"
    if guard:  # tests/test_engine.py:309-311
        monkeypatch.setattr(O, "REORTHO_THRESHOLD", -1.0)
    ad = pol.pop("adaptive", None)
    policy = PolicyConfig(**pol, adaptive=AdaptiveRankConfig(**ad) if ad else None)
    eng = OracleEngine(a0, k, reortho_guard=guard)
    recs = run_stream(eng, ev, policy, log_every)
    check_sim(golden, tag, sim_array(recs), n)
    if n is None:
        f = eng.factors
        np.testing.assert_allclose(f.s, golden[f"sim_{tag}_s"], rtol=1e-9)
        assert sine_angle(f.u, golden[f"sim_{tag}_u"]) < 1e-6
        assert sine_angle(f.vt.T, golden[f"sim_{tag}_vt"].T) < 1e-6
        assert abs(eng.sq_norm - float(golden[f"sim_{tag}_sq_norm"])) <= 1e-12 * eng.sq_norm


def _mixed_events(golden):
    kinds = golden["traj_mixed_kinds"]
    vecs = golden["traj_mixed_vecs"]
    m, n = golden["traj_mixed_a0"].shape
    ev, off = [], 0
    for k, i, j, d in kinds:
        if k == 0:
            ev.append(("row", vecs[off:off + n]))
            off += n
            m += 1
        elif k == 1:
            ev.append(("col", vecs[off:off + m]))
            off += m
            n += 1
        else:
            ev.append(("rank1", int(i), int(j), float(d)))
    return ev


def test_mixed_trajectory(golden):
    recs, eng = _trajectory(golden["traj_mixed_a0"], _mixed_events(golden), 6)
    _check_traj(golden, "mixed", recs, eng)


@pytest.mark.parametrize("b", [0, 1])
def test_cfg5a_streams(golden, b):
    a0, ev = workloads.cfg5a_stream(0, b, n_events=1024)
    eng = OracleEngine(a0, 32)
    for e in ev:
        if e[0] == "row":
            eng.row_append(e[1])
        else:
            eng.rank_one_update(e[1], e[2], e[3])
    assert rel_err(eng.factors.s, golden[f"s5a_{b}_s"]) < 1e-9
    assert sine_angle(eng.factors.vt.T, golden[f"s5a_{b}_vt"].T) < 1e-6
    # canonical signs: the first 64 rows agree entrywise
    np.testing.assert_allclose(eng.factors.u[:64], golden[f"s5a_{b}_u"], atol=1e-8)
