"""Stream sharding across GPUs: sessions share nothing, so
streams are partitioned over ranks with no data-path collective.  The only
cross-rank traffic is timing plumbing: a barrier and the max over ranks of the
timed region (torch.distributed, NCCL on GPUs / gloo on CPU).

``run_sharded`` is the N > 1 driver bench.py uses for BASELINE configs[4]
(64 concurrent streams over 1/2/4/8 GPUs); the device work sits behind a
small backend interface so the same driver runs under gloo with a stub
backend in tests/test_sharding.py.
"""

from __future__ import annotations

from typing import Protocol


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


class ShardBackend(Protocol):
    """The device side of one rank: its sessions and their timed steps."""

    def open(self, stream_ids: list[int]) -> None: ...

    def warm(self, steps: int) -> None: ...

    def run_timed(self, steps: int) -> float:
        """``steps`` steps of every owned stream; device milliseconds."""
        ...

    def close(self) -> None: ...


def run_sharded(n_total: int, world: int, rank: int, backend: ShardBackend, steps: int,
                warmup: int, dist=None, device=None) -> dict:
    """Open this rank's share of ``n_total`` streams, warm up, then time
    ``steps`` steps of all of them between barriers; the job's time is the
    max over ranks and its throughput every stream's frames over that time."""
    mine = streams_for_rank(n_total, world, rank)
    backend.open(mine)
    try:
        backend.warm(warmup)
        if dist is not None and dist.is_available() and dist.is_initialized():
            dist.barrier()
        ms = backend.run_timed(steps) if mine else 0.0
        ms_max = max_over_ranks(ms, dist, device)
    finally:
        backend.close()
    frames = n_total * steps
    return {"streams": mine, "ms_rank": ms, "ms": ms_max,
            "fps": frames / (ms_max * 1e-3) if ms_max > 0 else 0.0,
            "per_stream_fps": steps / (ms_max * 1e-3) if ms_max > 0 else 0.0}
