"""The N>1 host path on CPU: world_size-2 gloo process group over 127.0.0.1
(the GPU path shards independent sequences, so the only cross-rank steps
are barrier, max-over-ranks timing and the result gather)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_1711_07999_b200 import shard


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    r = shard.from_env()
    dist = shard.init(r, backend="gloo")
    try:
        mine = list(shard.shard(7, r))
        shard.barrier(r)
        mx = shard.max_over_ranks([rank + 1.5, -rank], r)
        sm = shard.sum_over_ranks([len(mine)], r)
        got = shard.gather_to_root({"rank": rank, "items": mine}, r)
        q.put((rank, mine, mx.tolist(), sm.tolist(), got))
    finally:
        dist.destroy_process_group()


def test_shard_partitions():
    for n in range(0, 20):
        for world in range(1, 9):
            parts = [list(shard.shard(n, shard.Rank(k, world))) for k in range(world)]
            flat = [i for p in parts for i in p]
            assert flat == list(range(n))
            assert max(map(len, parts)) - min(map(len, parts)) <= 1


def test_single_rank_is_identity():
    r = shard.Rank()
    assert shard.init(r) is None
    assert shard.max_over_ranks([3.0], r).tolist() == [3.0]
    assert shard.gather_to_root("x", r) == ["x"]


@pytest.mark.timeout(120)
def test_two_rank_gloo():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(k, world, port, q)) for k in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        rank, mine, mx, sm, got = q.get(timeout=100)
        res[rank] = (mine, mx, sm, got)
    for p in procs:
        p.join(timeout=30)
        assert p.exitcode == 0
    assert res[0][0] == [0, 1, 2, 3] and res[1][0] == [4, 5, 6]
    for k in range(world):
        assert res[k][1] == [2.5, 0.0]
        assert res[k][2] == [7.0]
    assert res[0][3] == [{"rank": 0, "items": [0, 1, 2, 3]}, {"rank": 1, "items": [4, 5, 6]}]
    assert res[1][3] is None
