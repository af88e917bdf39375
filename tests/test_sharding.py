"""Multi-process (world_size 2, gloo, CPU) coverage of the N > 1 path: stream
sharding with no data-path collective, max-over-ranks timing, aggregate
throughput."""

import os
import socket

import pytest
import torch.multiprocessing as mp

from paper_2301_00750_b200.sharding import aggregate_fps, max_over_ranks, streams_for_rank


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
