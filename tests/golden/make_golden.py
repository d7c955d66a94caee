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

    a0, ev, _ = workloads.cfg1(0, n_events=120)
    trajectory(a0, ev, 10, "cfg1", "periodic", period=100)

    a0, ev, _ = workloads.cfg2(0, n_events=60)
    trajectory(a0, ev, 20, "cfg2", "error", gamma=1.05)

    a0, ev, _ = workloads.cfg3(0, t_total=352)
    trajectory(a0, ev, 5, "cfg3", "angle", theta=float(np.deg2rad(5.0)))

    # mixed small stream: rows, cols, rank-1 (tests/test_engine.py:290-306 shape)
    g = np.random.default_rng(12)
    a0 = g.standard_normal((30, 25))
    m, n = 30, 25
    ev = []
    for t in range(300):
        kind = int(g.integers(10))
        if kind == 0:
            ev.append(("row", g.standard_normal(n)))
            m += 1
        elif kind == 1:
            ev.append(("col", g.standard_normal(m)))
            n += 1
        else:
            ev.append(("rank1", int(g.integers(m)), int(g.integers(n)), float(g.normal(0, 0.05))))
    out["traj_mixed_a0"] = a0
    kinds = []
    vecs = []
    for e in ev:
        if e[0] == "rank1":
            kinds.append([2, e[1], e[2], e[3]])
            vecs.append(np.zeros(0))
        else:
            kinds.append([0 if e[0] == "row" else 1, 0, 0, 0.0])
            vecs.append(e[1])
    out["traj_mixed_kinds"] = np.array(kinds, dtype=np.float64)
    out["traj_mixed_vecs"] = np.concatenate(vecs)
    trajectory(a0, ev, 6, "mixed")

    # ---- 5a streams (two sampled streams, first 64 events)
    for b in (0, 1):
        a0, ev = workloads.cfg5a_stream(0, b, n_events=64)
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
