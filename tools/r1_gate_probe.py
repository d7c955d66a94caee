"""V / U orthogonality drift of long rank-1 streams near the structure gate
(the test_rank_one_orthogonality_near_the_structure_gate scenario), printed
every 250 ticks; run twice, with and without ISVD_RANK1_WARP=1, to compare
the CTA-per-core and the one-warp rank-1 kernels."""
import os
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2605_24514_b200 import BatchedSvdEngine, _lib  # noqa
import ctypes as C  # noqa

kappa = float(sys.argv[1]) if len(sys.argv) > 1 else 99.0
rng = np.random.default_rng(int(kappa))
m, n, k, T = 160, 96, 20, 2000
qu = np.linalg.qr(rng.standard_normal((m, k)))[0]
qv = np.linalg.qr(rng.standard_normal((n, k)))[0]
sig = np.geomspace(10.0, 10.0 / kappa, k)
a0 = (qu * sig) @ qv.T
B = 64
eng = BatchedSvdEngine(np.repeat(a0[None], B, axis=0), k)
ii, jj = rng.integers(0, m, T), rng.integers(0, n, T)
dd = rng.normal(0.0, 1e-3, T)
lib = _lib.load()
cnt = (C.c_int64 * 8)()
lib.isvd_debug_counters(cnt, 1)
tag = "warp" if os.environ.get("ISVD_RANK1_WARP") == "1" else "cta"
for t in range(T):
    eng.rank_one_update(np.full(B, ii[t]), np.full(B, jj[t]), np.full(B, dd[t]))
    if (t + 1) % 250 == 0:
        du, dv = eng.ortho_defect()
        eng.synchronize()
        lib.isvd_debug_counters(cnt, 0)
        print(f"{tag} kappa={kappa} t={t + 1} du={np.max(du):.2e} dv={np.max(dv):.2e} cores={cnt[1]} "
              f"fast={cnt[7]} steps={cnt[6]} sweeps={cnt[0]}", flush=True)
