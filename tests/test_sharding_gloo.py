"""N > 1 host path of the batched-stream benchmark on CPU: world_size 2 over
the gloo backend (the GPU run uses the same code over NCCL)."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2605_24514_b200.sharding import max_over_ranks, shard_streams, sum_over_ranks


def test_shards_partition_streams():
    for total in (4096, 4097, 10):
        for world in (1, 2, 3, 4, 8):
            if total < world:
                continue
            ids = [i for r in range(world) for i in shard_streams(total, world, r)]
            assert ids == list(range(total))
            sizes = [len(shard_streams(total, world, r)) for r in range(world)]
            assert max(sizes) - min(sizes) <= 1


def test_shard_validation():
    with pytest.raises(ValueError):
        shard_streams(10, 2, 2)
    with pytest.raises(ValueError):
        shard_streams(1, 2, 0)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import OracleEngine
        from paper_2605_24514_b200 import workloads

        mine = shard_streams(8, world, rank)
        # every rank runs its streams' first events through the CPU oracle;
        # the per-stream result must not depend on which rank ran it
        sig = {}
        for b in mine:
            a0, ev = workloads.cfg5a_stream(0, b, m=64, n=32, rank=4, n_events=6)
            e = OracleEngine(a0, 4)
            for x in ev:
                if x[0] == "row":
                    e.row_append(x[1])
                else:
                    e.rank_one_update(x[1], x[2], x[3])
            sig[b] = float(e.factors.s[0])
        t_local = 1.0 + rank  # stand-in for the timed region length
        out[rank] = (list(mine), sig, max_over_ranks(t_local), sum_over_ranks(len(mine)))
        dist.barrier()
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_sharding_and_max_timing():
    world = 2
    port = _free_port()
    manager = mp.Manager()
    out = manager.dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    ranks = dict(out)
    assert set(ranks) == {0, 1}
    owned = ranks[0][0] + ranks[1][0]
    assert sorted(owned) == list(range(8))
    assert ranks[0][2] == ranks[1][2] == 2.0          # max over ranks
    assert ranks[0][3] == ranks[1][3] == 8.0          # all streams processed
    # world-size independence: stream 5 computed on its own gives the same result
    from oracle import OracleEngine
    from paper_2605_24514_b200 import workloads

    a0, ev = workloads.cfg5a_stream(0, 5, m=64, n=32, rank=4, n_events=6)
    e = OracleEngine(a0, 4)
    for x in ev:
        if x[0] == "row":
            e.row_append(x[1])
        else:
            e.rank_one_update(x[1], x[2], x[3])
    got = {**ranks[0][1], **ranks[1][1]}
    assert got[5] == float(e.factors.s[0])
