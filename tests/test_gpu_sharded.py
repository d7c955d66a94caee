"""Row-sharded tall stream (BASELINE config 5b) on the GPU.

Two ranks (torch.distributed gloo, both on cuda:0 -- the kernels of the two
processes never wait on each other; the cross-rank sums go through the host)
run ShardedSvdEngine over a row-split matrix; the gathered result must match
one unsharded engine on the whole matrix: sigma within 1e-9 relative, sine
subspace angles < 1e-6, the tracked squared norm, residuals and metrics.
"""

import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from conftest import rel_err, sine_angle

pytestmark = pytest.mark.gpu

M, N, K = 24000, 256, 32


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _problem(seed=3):
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((M, K))
    y = rng.standard_normal((N, K))
    a0 = x @ y.T + 0.05 * rng.standard_normal((M, N))
    rows = rng.standard_normal((40, K)) @ y.T + 0.05 * rng.standard_normal((40, N))
    rows = np.hstack([rows, 0.05 * rng.standard_normal((40, 2))])  # entries of appended columns
    cols = rng.standard_normal((3, M + 40))
    return a0, rows, cols


def _events():
    """A mixed sequence: 20 rows, a column, rank-1s in both shards and in an
    appended row, more rows, a column, a refresh-free tail."""
    ev = [("row", t) for t in range(20)]
    ev += [("col", 0), ("r1", (5, 7, 0.3)), ("r1", (M - 3, 100, -0.2)), ("r1", (M + 4, 3, 0.5))]
    ev += [("row", t) for t in range(20, 40)]
    ev += [("col", 1), ("r1", (M // 2, 255, 0.1))]
    return ev


def _worker(rank, world, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    from paper_2605_24514_b200.sharded import ShardedSvdEngine, shard_rows

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    a0, rows, cols = _problem()
    r0, ml = shard_rows(M, world, rank)
    eng = ShardedSvdEngine(a0[r0:r0 + ml], K, m_global=M, row0=r0, rows_cap=M + 64)
    rec = {"s0": eng.factors.s.copy()}
    m_now, n_now = M, N
    for kind, arg in _events():
        if kind == "row":
            eng.row_append(rows[arg][:n_now])
            m_now += 1
        elif kind == "col":
            eng.col_append(cols[arg][:m_now])
            n_now += 1
        else:
            eng.rank_one_update(*arg)
    f = eng.gather_factors()
    sq, rho, xn = eng.scalars()
    du, dv = eng.ortho_defect()
    fe = eng.frob_error()
    if rank == 0:
        np.savez(os.path.join(out_dir, "sharded.npz"), u=f.u, s=f.s, vt=f.vt, sq=sq, rho=rho,
                 xn=xn, du=du, dv=dv, fe=fe, s0=rec["s0"], shape=np.array(eng.shape))
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_matches_unsharded():
    from paper_2605_24514_b200 import SvdEngine
    from paper_2605_24514_b200.linalg import orthonormality_defect

    with tempfile.TemporaryDirectory() as d:
        mp.start_processes(_worker, args=(2, _free_port(), d), nprocs=2, join=True,
                           start_method="spawn")
        got = dict(np.load(os.path.join(d, "sharded.npz")))
    a0, rows, cols = _problem()
    ref = SvdEngine(a0, K, capacity=(M + 64, N + 8, K))
    s0 = ref.factors.s.copy()
    m_now, n_now = M, N
    for kind, arg in _events():
        if kind == "row":
            ref.row_append(rows[arg][:n_now])
            m_now += 1
        elif kind == "col":
            ref.col_append(cols[arg][:m_now])
            n_now += 1
        else:
            ref.rank_one_update(*arg)
    f = ref.factors
    assert tuple(got["shape"]) == ref.shape
    assert rel_err(got["s0"], s0) < 1e-9
    assert rel_err(got["s"], f.s) < 1e-9
    assert sine_angle(got["u"], f.u) < 1e-6
    assert sine_angle(got["vt"].T, f.vt.T) < 1e-6
    assert orthonormality_defect(got["u"]) < 1e-9
    assert abs(float(got["sq"]) - ref.sq_norm) <= 1e-12 * ref.sq_norm
    assert abs(float(got["rho"]) - ref.last_residual) <= 1e-8 * max(1.0, ref.last_input_norm)
    # same sign convention (column max |u| non-negative) as the unsharded engine
    lead = np.argmax(np.abs(got["u"]), axis=0)
    assert np.all(got["u"][lead, np.arange(got["u"].shape[1])] >= 0.0)
    np.testing.assert_allclose(got["u"], f.u, atol=1e-8)
    from paper_2605_24514_b200 import frob_error
    assert abs(float(got["fe"]) - frob_error(ref)) <= 1e-9 * max(1.0, frob_error(ref))
    assert float(got["du"]) < 1e-9 and float(got["dv"]) < 1e-9
