"""Row-sharded tall-stream algorithm on CPU, world_size 2 over gloo.

The numpy model in tests/sharded_model.py follows the CUDA shard mode step
by step (which sums cross ranks, what is replicated, which rank stores the
appended rows); gathered over two gloo ranks it must reproduce the unsharded
reference restatement (oracle/) on the same events.  The GPU run of the real
engine is tests/test_gpu_sharded.py."""

import os
import socket
import tempfile

import numpy as np
import torch
import torch.multiprocessing as mp

from conftest import rel_err, sine_angle
from paper_2605_24514_b200.sharded import shard_rows

M, N, K = 300, 40, 6


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _problem():
    rng = np.random.default_rng(11)
    a0 = rng.standard_normal((M, K)) @ rng.standard_normal((K, N)) + 0.05 * rng.standard_normal((M, N))
    rows = rng.standard_normal((12, N + 2))
    cols = rng.standard_normal((2, M + 12))
    return a0, rows, cols


EVENTS = ([("row", t) for t in range(6)] + [("col", 0), ("r1", (3, 5, 0.4)),
          ("r1", (M + 2, 7, -0.3)), ("r1", (M // 2 + 1, 0, 0.2))] +
          [("row", t) for t in range(6, 12)] + [("col", 1)])


def _run(eng, rows, cols):
    m_now, n_now = M, N
    for kind, arg in EVENTS:
        if kind == "row":
            eng.row_append(rows[arg][:n_now])
            m_now += 1
        elif kind == "col":
            eng.col_append(cols[arg][:m_now])
            n_now += 1
        else:
            eng.rank_one_update(*arg)


def _worker(rank, world, port, out_dir):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from sharded_model import ShardModel

    def allreduce(x):
        t = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64)).clone()
        dist.all_reduce(t)
        return t.numpy()

    a0, rows, cols = _problem()
    r0, ml = shard_rows(M, world, rank)
    eng = ShardModel(a0[r0:r0 + ml], K, M, r0, rank, world, allreduce)
    _run(eng, rows, cols)
    blocks = [None] * world
    dist.all_gather_object(blocks, eng.u)
    if rank == 0:
        np.savez(os.path.join(out_dir, "model.npz"), u=np.vstack(blocks), s=eng.s, vt=eng.vt,
                 sq=eng.sq)
    dist.barrier()
    dist.destroy_process_group()


def test_shard_rows_partition():
    for m in (1, 7, 300, 4194304):
        for world in (1, 2, 3, 8):
            if m < world:
                continue
            blocks = [shard_rows(m, world, r) for r in range(world)]
            assert blocks[0][0] == 0
            for (a, la), (b, _) in zip(blocks, blocks[1:]):
                assert a + la == b
            assert blocks[-1][0] + blocks[-1][1] == m
            assert max(b[1] for b in blocks) - min(b[1] for b in blocks) <= 1


def test_sharded_model_matches_oracle_gloo():
    from oracle import OracleEngine

    with tempfile.TemporaryDirectory() as d:
        mp.start_processes(_worker, args=(2, _free_port(), d), nprocs=2, join=True,
                           start_method="spawn")
        got = dict(np.load(os.path.join(d, "model.npz")))
    a0, rows, cols = _problem()
    ref = OracleEngine(a0, K)
    _run(ref, rows, cols)
    f = ref.factors
    assert got["u"].shape == f.u.shape
    assert rel_err(got["s"], f.s) < 1e-9
    assert sine_angle(got["u"], f.u) < 1e-6
    assert sine_angle(got["vt"].T, f.vt.T) < 1e-6
    np.testing.assert_allclose(got["u"], f.u, atol=1e-8)  # same canonical signs
    assert abs(float(got["sq"]) - ref.sq_norm) <= 1e-12 * ref.sq_norm
