"""Ad-hoc GPU sanity script (not a test): exercises each C-ABI entry point on
small inputs and prints the deviation from the numpy oracle."""

import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from oracle import (OracleEngine, core_svd_jacobi, full_svd as o_full_svd, kernel_rank_one,  # noqa
                    kernel_row_append, sine_angle_max)
from paper_2605_24514_b200 import SvdEngine, BatchedSvdEngine, full_svd  # noqa
from paper_2605_24514_b200 import _lib  # noqa


def rel(a, b):
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-300)))


def main():
    import torch

    lib = _lib.load()
    rng = np.random.default_rng(1)
    # core svd
    for s in (1, 2, 5, 17, 33, 65, 129):
        cores = rng.standard_normal((4, s, s))
        dc = torch.tensor(cores, device="cuda")
        u = torch.empty_like(dc)
        vt = torch.empty_like(dc)
        sv = torch.empty((4, s), dtype=torch.float64, device="cuda")
        _lib.check(lib.isvd_core_svd(4, s, dc.data_ptr(), u.data_ptr(), sv.data_ptr(), vt.data_ptr(), None))
        torch.cuda.synchronize()
        un, svn, vtn = u.cpu().numpy(), sv.cpu().numpy(), vt.cpu().numpy()
        err = max(np.max(np.abs((un[b] * svn[b]) @ vtn[b] - cores[b])) for b in range(4))
        ref = [np.linalg.svd(cores[b], compute_uv=False) for b in range(4)]
        print(f"core_svd s={s}: recon {err:.2e}  sigma rel {max(rel(svn[b], ref[b]) for b in range(4)):.2e}")
    # dense svd
    for (m, n) in ((2, 2), (9, 7), (7, 9), (200, 100), (1024, 256), (100, 300)):
        a = rng.standard_normal((m, n))
        t0 = time.perf_counter()
        f = full_svd(a)
        dt = time.perf_counter() - t0
        fo = o_full_svd(a)
        print(f"full_svd {m}x{n}: sigma rel {rel(f.s, fo.s):.2e} recon {np.max(np.abs((f.u*f.s)@f.vt - a)):.2e} "
              f"ortho {np.linalg.norm(f.u.T@f.u-np.eye(f.u.shape[1])):.2e} signs {np.max(np.abs(f.u-fo.u)):.2e} t={dt*1e3:.1f}ms")
    # engine
    a0 = rng.standard_normal((60, 6)) @ rng.standard_normal((6, 40)) + 0.05 * rng.standard_normal((60, 40))
    g = SvdEngine(a0, 6)
    c = OracleEngine(a0, 6)
    for t in range(200):
        k = t % 3
        if k == 0:
            x = rng.standard_normal(g.shape[1]); g.row_append(x); c.row_append(x)
        elif k == 1:
            y = rng.standard_normal(g.shape[0]); g.col_append(y); c.col_append(y)
        else:
            i, j, d = int(rng.integers(g.shape[0])), int(rng.integers(g.shape[1])), float(rng.normal(0, .1))
            g.rank_one_update(i, j, d); c.rank_one_update(i, j, d)
    print("engine mixed 200: s rel", rel(g.factors.s, c.factors.s), "angle",
          sine_angle_max(g.factors.u, c.factors.u), "sign-match", np.max(np.abs(g.factors.u - c.factors.u)),
          "sqnorm", g.sq_norm - c.sq_norm, "tracked", np.max(np.abs(g.tracked - c.tracked)))
    # batched 5a small
    from paper_2605_24514_b200 import workloads
    a0b, ticks, streams = workloads.cfg5a_batch(0, 4, n_events=32)
    be = BatchedSvdEngine(a0b, 32, m_cap=1100)
    for tk in ticks:
        if tk[0] == "row":
            be.row_append(tk[1])
        else:
            be.rank_one_update(tk[1], tk[2], tk[3])
    for b in range(4):
        oe = OracleEngine(streams[b][0], 32)
        for e in streams[b][1]:
            if e[0] == "row":
                oe.row_append(e[1])
            else:
                oe.rank_one_update(e[1], e[2], e[3])
        f = be.factors(b)
        print(f"5a stream {b}: s rel {rel(f.s, oe.factors.s):.2e} angle {sine_angle_max(f.u, oe.factors.u):.2e}")


if __name__ == "__main__":
    main()
