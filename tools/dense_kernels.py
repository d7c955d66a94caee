"""Time the dense contractions of the refresh / oracle / metrics path at
BASELINE config 4's final size (25000 x 6000, rank-64 geometric spectrum +
N(0, 0.01^2), k = 64): engine init (truncated SVD), the full-SVD oracle
(compute_oracle on the resident tracked matrix) and frob_error.

  python tools/dense_kernels.py [m n] [--once]     (--once: one of each, for ncu)
"""
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2605_24514_b200 import SvdEngine, compute_oracle, frob_error, workloads  # noqa

args = [a for a in sys.argv[1:] if not a.startswith("--")]
once = "--once" in sys.argv
m, n = (int(args[0]), int(args[1])) if len(args) >= 2 else (25_000, 6_000)
a0, _, _ = workloads.cfg4(m=m, n=n, n_blocks=0)


def timed(f):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = f()
    torch.cuda.synchronize()
    return r, time.perf_counter() - t0


eng, t_init = timed(lambda: SvdEngine(a0, k=64))
out = {"shape": [m, n], "k": 64, "init_s": t_init}
reps = 1 if once else 2
out["oracle_s"] = [timed(lambda: compute_oracle(eng, 64))[1] for _ in range(reps)]
fe = [timed(lambda: frob_error(eng)) for _ in range(1 if once else 3)]
out["frob_error_s"] = [t for _, t in fe]
out["frob_error"] = fe[0][0]
if not once:
    o = compute_oracle(eng, 64)
    out["frob_opt"] = o.frob_opt
    out["ratio"] = fe[0][0] / o.frob_opt
    # cross-check against LAPACK on the host (the reference's np.linalg.svd)
    t0 = time.perf_counter()
    s_ref = np.linalg.svd(a0, compute_uv=False)
    out["lapack_s"] = time.perf_counter() - t0
    out["sigma_rel_err_top64"] = float(np.max(np.abs(o.singular_values[:64] - s_ref[:64]) / s_ref[:64]))
    tail = np.sqrt(np.sum(s_ref[64:] ** 2))
    out["frob_opt_rel_err"] = abs(o.frob_opt - tail) / tail
    rec = (eng.factors.u * eng.factors.s) @ eng.factors.vt
    direct = float(np.linalg.norm(a0 - rec))
    out["frob_error_rel_err"] = abs(fe[0][0] - direct) / direct
print(json.dumps(out, indent=1))
