"""Generate golden vectors from the REAL reference (svdstream) -- run here only.

    python tests/golden/make_golden.py

Imports the reference from /root/reference/pkg/src (read-only).  When
Cython is available, the reference's compiled Jacobi backend
(_kernels.pyx) is built in a scratch copy under /tmp so both reference
backends contribute fixtures.  Outputs small .npz files next to this script;
they are committed, and the GPU box never needs /root/reference.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
import tempfile
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REPO = HERE.parent.parent
sys.path.insert(0, str(REPO))

from paper_2605_24514_b200 import workloads  # noqa: E402

REF_PKG = Path("/root/reference/pkg")


def _import_reference():
    """Scratch copy of the reference with its Cython kernel compiled in place."""
    scratch = Path(tempfile.mkdtemp(prefix="svdstream_ref_"))
    shutil.copytree(REF_PKG / "src", scratch / "src")
    src = scratch / "src" / "svdstream"
    try:
        subprocess.run([sys.executable, "-m", "cython", "-3", "--fast-fail", str(src / "_kernels.pyx")],
                       check=True, capture_output=True)
        import sysconfig

        inc = sysconfig.get_paths()["include"]
        npinc = np.get_include()
        ext = sysconfig.get_config_var("EXT_SUFFIX")
        subprocess.run(["gcc", "-O3", "-shared", "-fPIC", f"-I{inc}", f"-I{npinc}",
                        str(src / "_kernels.c"), "-o", str(src / f"_kernels{ext}")],
                       check=True, capture_output=True)
    except Exception as exc:  # pragma: no cover - best effort
        print("compiled backend unavailable:", exc)
    sys.path.insert(0, str(scratch / "src"))
    import svdstream

    return svdstream


def _mixed_stream(g, m, n, count):
    """Random mix: 10 % row appends, 10 % column appends, 80 % rank-1."""
    ev = []
    for _ in range(count):
        kind = int(g.integers(10))
        if kind == 0:
            ev.append(("row", g.standard_normal(n)))
            m += 1
        elif kind == 1:
            ev.append(("col", g.standard_normal(m)))
            n += 1
        else:
            ev.append(("rank1", int(g.integers(m)), int(g.integers(n)), float(g.normal(0, 0.05))))
    return ev


def _encode_events(ev):
    kinds, vecs = [], []
    for e in ev:
        if e[0] == "rank1":
            kinds.append([2, e[1], e[2], e[3]])
        else:
            kinds.append([0 if e[0] == "row" else 1, 0, 0, 0.0])
            vecs.append(e[1])
    return np.array(kinds, dtype=np.float64), np.concatenate(vecs) if vecs else np.zeros(0)


def main():
    sv = _import_reference()
    from svdstream import backend
    from svdstream.engine import SvdEngine
    from svdstream import metrics as M
    from svdstream.linalg import full_svd

    print("reference backends:", backend.available_backends())
    out = {}

    # ---- core_svd known answers / random cores, both backends
    rng = np.random.default_rng(2024)
    cores = {f"rand{s}": rng.standard_normal((s, s)) for s in (1, 2, 5, 9, 16, 33)}
    cores["dead"] = np.array([[3.0, 1.0], [0.0, 0.0]])
    # a Brand row-append core: [[diag s, 0], [p, rho]]
    s = np.sort(np.abs(rng.standard_normal(32)) * 10)[::-1]
    brand = np.zeros((33, 33))
    brand[np.arange(32), np.arange(32)] = s
    brand[32, :32] = rng.standard_normal(32)
    brand[32, 32] = 0.7
    cores["brand33"] = brand
    for name in backend.available_backends():
        backend.set_backend(name)
        for key, c in cores.items():
            u, sv_, vt = backend.core_svd(c)
            out[f"core_{name}_{key}_in"] = c
            out[f"core_{name}_{key}_s"] = sv_
            out[f"core_{name}_{key}_recon"] = (u * sv_) @ vt
    backend.set_backend("auto")

    # ---- kernel contracts (row_append, rank_one) on random factors
    def rand_factors(m, n, r, seed):
        g = np.random.default_rng(seed)
        f = full_svd(g.standard_normal((m, r)) @ g.standard_normal((r, n)))
        return f.u[:, :r].copy(), f.s[:r].copy(), f.vt[:r, :].copy()

    u, s_, vt = rand_factors(10, 8, 4, 99)
    x = np.random.default_rng(7).standard_normal(8)
    for name in backend.available_backends():
        backend.set_backend(name)
        u2, s2, vt2, rho = backend.row_append(u, s_, vt, x, 1e-10, 5)
        out[f"ra_{name}_s"] = s2
        out[f"ra_{name}_recon"] = (u2 * s2) @ vt2
        out[f"ra_{name}_rho"] = np.array(rho)
        u3, s3, vt3 = backend.rank_one(u, s_, vt, 3, 6, 0.25, 4)
        out[f"r1_{name}_s"] = s3
        out[f"r1_{name}_recon"] = (u3 * s3) @ vt3
    backend.set_backend("auto")
    out["ra_in_u"], out["ra_in_s"], out["ra_in_vt"], out["ra_in_x"] = u, s_, vt, x

    # ---- engine trajectories on BASELINE-shaped streams (shortened)
    def trajectory(a0, events, k, tag, policy_kind=None, period=None, gamma=None, theta=None):
        eng = SvdEngine(a0, k)
        eng.set_reference()
        recs = []
        t_last = 0
        for t, ev in enumerate(events, start=1):
            if ev[0] == "row":
                eng.row_append(ev[1])
            elif ev[0] == "col":
                eng.col_append(ev[1])
            else:
                eng.rank_one_update(ev[1], ev[2], ev[3])
            orc = M.compute_oracle(eng.tracked, eng.work_rank)
            fire = False
            if policy_kind == "periodic":
                fire = t % period == 0
            elif policy_kind == "error":
                r = M.error_ratio(M.frob_error(eng), orc.frob_opt)
                fire = (not np.isnan(r)) and r > gamma
            elif policy_kind == "angle":
                fire = M.angle_to_opt(eng, orc.basis) > theta
            if fire:
                eng.refresh(store_reference=True)
                t_last = t
            rec = M.collect(eng, 0.0, fire, orc)
            recs.append([rec.frob_error, rec.evr, rec.rank, float(rec.refreshed), rec.frob_opt,
                         rec.frob_ratio if rec.frob_ratio is not None else np.nan,
                         rec.angle_opt])
        f = eng.factors
        out[f"traj_{tag}_records"] = np.array(recs, dtype=np.float64)
        out[f"traj_{tag}_s"] = f.s
        out[f"traj_{tag}_u"] = f.u
        out[f"traj_{tag}_vt"] = f.vt
        out[f"traj_{tag}_sq_norm"] = np.array(eng.sq_norm)

    # ---- whole BASELINE streams through the reference's OWN loop
    # (stream.run_simulation, stream.py:257-333), fed our seeded inputs by
    # replacing its two generator hooks (gen_low_rank, build_events).
    import svdstream.engine as ref_engine
    import svdstream.stream as S
    from svdstream.policies import AdaptiveRankConfig, PolicyConfig

    def simulate(tag, a0, events, k, policy, log_every, reortho_guard=False):
        ref_events = [S.RowAppend(e[1]) if e[0] == "row" else S.ColAppend(e[1]) if e[0] == "col"
                      else S.RankOneUpdate(e[1], e[2], e[3]) for e in events]
        gen0, build0 = S.gen_low_rank, S.build_events
        S.gen_low_rank = lambda *a, **kw: np.array(a0, dtype=np.float64, copy=True)
        S.build_events = lambda spec: ref_events
        try:
            spec = S.StreamSpec(m=a0.shape[0], n=a0.shape[1], true_rank=1, k=k,
                                events=len(events), policy=policy, log_every=log_every,
                                reortho_guard=reortho_guard)
            recs, eng = S.run_simulation(spec, return_engine=True)
        finally:
            S.gen_low_rank, S.build_events = gen0, build0
        nan = lambda v: np.nan if v is None else float(v)
        out[f"sim_{tag}_records"] = np.array(
            [[r.step, r.frob_error, r.evr, r.rank, float(r.refreshed), nan(r.frob_opt),
              nan(r.frob_ratio), nan(r.angle_ref), nan(r.angle_opt)] for r in recs])
        f = eng.factors
        out[f"sim_{tag}_s"] = f.s
        out[f"sim_{tag}_u"] = f.u
        out[f"sim_{tag}_vt"] = f.vt
        out[f"sim_{tag}_sq_norm"] = np.array(eng.sq_norm)
        r = out[f"sim_{tag}_records"]
        print(f"  {tag}: {len(recs)} records, refreshes {int(np.nansum(r[:, 4]))}, "
              f"ranks {sorted(set(r[:, 3].astype(int).tolist()))}")

    # config 1: all 1000 row appends, periodic 100, oracle every tick
    a0, ev, _ = workloads.cfg1(0, n_events=1000)
    simulate("cfg1", a0, ev, 10, PolicyConfig(kind="periodic", period=100), 1)
    # config 2: 2000 of the 10,000 rank-1 updates, error trigger 1.05, oracle every tick
    a0, ev, _ = workloads.cfg2(0, n_events=2000)
    simulate("cfg2", a0, ev, 20, PolicyConfig(kind="error", gamma=1.05, min_spacing=0), 1)
    # config 3: all 2268 daily appends, angle trigger 5 deg, oracle every tick
    a0, ev, _ = workloads.cfg3(0)
    simulate("cfg3", a0, ev, 5, PolicyConfig(kind="angle", theta_max=float(np.deg2rad(5.0))), 1)
    # config 4 at reduced size, same code path: sigma_i = 0.9^i rank 64, 5 rows : 1 col,
    # k0 = 64, adaptive rank (EVR 0.95, k_max 128, novelty eta 0.5), periodic refresh 200,
    # oracle every 50 ticks (4 observations per refresh for the two-step hysteresis)
    a0, ev, _ = workloads.cfg4(0, m=400, n=120, rank=64, n_blocks=200)
    simulate("cfg4r", a0, ev, 64,
             PolicyConfig(kind="periodic", period=200,
                          adaptive=AdaptiveRankConfig(tau=0.95, k_min=1, k_max=128, eta=0.5)), 50)
    # the same with a rank floor high enough for the novelty bump to fire
    simulate("cfg4b", a0, ev[:600], 12,
             PolicyConfig(kind="periodic", period=150,
                          adaptive=AdaptiveRankConfig(tau=0.99, k_min=4, k_max=40, eta=0.05)), 25)
    # reortho guard forced on every tick (tests/test_engine.py:309-323 monkeypatches the
    # threshold the same way), on the mixed stream below
    guard_events = _mixed_stream(np.random.default_rng(13), 40, 30, 240)
    thr0 = ref_engine.REORTHO_THRESHOLD
    ref_engine.REORTHO_THRESHOLD = -1.0
    try:
        g0 = np.random.default_rng(14).standard_normal((40, 30))
        out["sim_guard_a0"] = g0
        out["sim_guard_kinds"], out["sim_guard_vecs"] = _encode_events(guard_events)
        simulate("guard", g0, guard_events, 6, PolicyConfig(kind="periodic", period=80), 10,
                 reortho_guard=True)
    finally:
        ref_engine.REORTHO_THRESHOLD = thr0

    # mixed small stream: rows, cols, rank-1 (tests/test_engine.py:290-306 shape)
    g = np.random.default_rng(12)
    a0 = g.standard_normal((30, 25))
    ev = _mixed_stream(g, 30, 25, 300)
    out["traj_mixed_a0"] = a0
    out["traj_mixed_kinds"], out["traj_mixed_vecs"] = _encode_events(ev)
    trajectory(a0, ev, 6, "mixed")

    # ---- 5a streams (two sampled streams, all 1024 events)
    for b in (0, 1):
        a0, ev = workloads.cfg5a_stream(0, b, n_events=1024)
        eng = SvdEngine(a0, 32)
        for e in ev:
            if e[0] == "row":
                eng.row_append(e[1])
            else:
                eng.rank_one_update(e[1], e[2], e[3])
        out[f"s5a_{b}_s"] = eng.factors.s
        out[f"s5a_{b}_u"] = eng.factors.u[:64]
        out[f"s5a_{b}_vt"] = eng.factors.vt

    np.savez_compressed(HERE / "reference_golden.npz", **out)
    sizes = sum(v.nbytes for v in out.values())
    print(f"wrote {len(out)} arrays, {sizes / 1e6:.1f} MB raw")


if __name__ == "__main__":
    main()
