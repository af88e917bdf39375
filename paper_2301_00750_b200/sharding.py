"""Stream sharding across GPUs: sessions share nothing, so
streams are partitioned over ranks with no data-path collective.  The only
cross-rank traffic is timing plumbing: a barrier and the max over ranks of the
timed region (torch.distributed, NCCL on GPUs / gloo on CPU)."""

from __future__ import annotations


def streams_for_rank(n_streams: int, world: int, rank: int) -> list[int]:
    """Stream ids owned by ``rank``: stream i -> rank i mod world."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("invalid rank / world size")
    return list(range(rank, n_streams, world))


def max_over_ranks(value: float, dist=None, device=None) -> float:
    """The job's time is the slowest rank's (timings are never wall-clock
    across processes)."""
    if dist is None or not dist.is_available() or not dist.is_initialized():
        return float(value)
    import torch

    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def aggregate_fps(frames_per_rank: int, world: int, seconds_max: float) -> float:
    """Whole-job throughput: every rank processed ``frames_per_rank`` frames
    in at most ``seconds_max``."""
    return world * frames_per_rank / seconds_max
