"""Multi-GPU plumbing for the batched-stream workload (BASELINE config 5a).

Streams are independent units: each rank owns a contiguous
block of stream ids and runs its own engine; the only communication is a
barrier and a max-over-ranks reduction of the timed region (no data-path
collective).  Per-stream inputs are seeded by the global stream id, so a
stream's data does not depend on the world size.
"""

from __future__ import annotations


def shard_streams(total: int, world: int, rank: int) -> range:
    """Contiguous block of stream ids owned by ``rank`` (sizes differ by <= 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} for world size {world}")
    if total < world:
        raise ValueError(f"{total} streams cannot be split over {world} ranks")
    base, extra = divmod(total, world)
    start = rank * base + min(rank, extra)
    return range(start, start + base + (1 if rank < extra else 0))


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank scalar (timed-region length) over the process group;
    identity when torch.distributed is not initialised."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()):
        return float(value)
    if dist.get_backend() != "nccl":
        device = None  # gloo reduces host tensors
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(value: float, device=None) -> float:
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()):
        return float(value)
    if dist.get_backend() != "nccl":
        device = None
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())
