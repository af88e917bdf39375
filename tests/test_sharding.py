"""Multi-process (world_size 2, gloo, CPU) coverage of the N > 1 path: stream
sharding with no data-path collective, max-over-ranks timing, aggregate
throughput."""

import os
import socket

import pytest
import torch.multiprocessing as mp

from paper_2301_00750_b200.sharding import (aggregate_fps, max_over_ranks, run_sharded,
                                            streams_for_rank)


def test_partition_is_disjoint_and_complete():
    for world in (1, 2, 4, 8):
        owned = [streams_for_rank(64, world, r) for r in range(world)]
        flat = sorted(s for o in owned for s in o)
        assert flat == list(range(64))
        assert all(len(o) == 64 // world for o in owned)
    with pytest.raises(ValueError):
        streams_for_rank(4, 2, 2)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    mine = streams_for_rank(6, world, rank)
    elapsed = 1.0 + rank  # rank 1 is the slow one
    slowest = max_over_ranks(elapsed, dist)
    out[rank] = (mine, slowest, aggregate_fps(len(mine) * 10, world, slowest))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo_timing_and_sharding():
    mgr = mp.Manager()
    out = mgr.dict()
    port = _free_port()
    mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
    assert out[0][0] == [0, 2, 4] and out[1][0] == [1, 3, 5]
    assert out[0][1] == out[1][1] == 2.0          # max over ranks
    assert out[0][2] == pytest.approx(2 * 30 / 2.0)


class _StubBackend:
    """Stands in for bench.ThreadedSessions (the GPU sessions): records what
    the driver asks for; rank r's timed region takes 10 * (r + 1) ms."""

    def __init__(self, rank):
        self.rank, self.calls = rank, []

    def open(self, ids):
        self.calls.append(("open", list(ids)))

    def warm(self, steps):
        self.calls.append(("warm", steps))

    def run_timed(self, steps):
        self.calls.append(("timed", steps))
        return 10.0 * (self.rank + 1)

    def close(self):
        self.calls.append(("close",))


def _driver_worker(rank, world, port, out):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    be = _StubBackend(rank)
    r = run_sharded(64, world, rank, be, steps=5, warmup=2, dist=dist)
    out[rank] = (r, be.calls)
    dist.destroy_process_group()


def test_run_sharded_two_ranks_gloo():
    """The driver bench.py uses for configs[4] (64 streams over N GPUs), under
    gloo with a stub device layer: disjoint halves of the streams, one warm-up
    and one timed region per rank, the job time is the slowest rank's, and the
    throughput counts every stream's frames."""
    mgr = mp.Manager()
    out = mgr.dict()
    port = _free_port()
    mp.spawn(_driver_worker, args=(2, port, out), nprocs=2, join=True)
    (r0, c0), (r1, c1) = out[0], out[1]
    assert r0["streams"] == list(range(0, 64, 2)) and r1["streams"] == list(range(1, 64, 2))
    assert c0 == [("open", r0["streams"]), ("warm", 2), ("timed", 5), ("close",)]
    assert r0["ms"] == r1["ms"] == 20.0  # max over ranks
    assert r0["fps"] == pytest.approx(64 * 5 / 0.020)
    assert r0["per_stream_fps"] == pytest.approx(5 / 0.020)


def test_run_sharded_single_rank_no_dist():
    be = _StubBackend(0)
    r = run_sharded(8, 1, 0, be, steps=3, warmup=1)
    assert r["streams"] == list(range(8)) and r["ms"] == 10.0
    assert r["fps"] == pytest.approx(8 * 3 / 0.010)
