"""The PDQ unit sharding / exchange protocol over world_size 2 with gloo on
CPU (the production path runs the same collectives over NCCL)."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2503_22227_b200.pdq.shard import ShardGroup

    g = ShardGroup.from_env()
    calls = []

    def fn(u):
        calls.append(u)
        base = torch.arange(6, dtype=torch.int64) * (u + 1)
        return (base, None if u % 2 else base * 3)

    res = g.map_units(list(range(7)), fn)
    out[rank] = {"calls": calls, "res": [(r[0].tolist(), None if r[1] is None else r[1].tolist())
                                          for r in res]}
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_units_split_and_exchanged(world):
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    want = [([v * (u + 1) for v in range(6)],
             None if u % 2 else [3 * v * (u + 1) for v in range(6)]) for u in range(7)]
    seen = []
    for r in range(world):
        assert out[r]["res"] == want
        assert out[r]["calls"] == [u for u in range(7) if u % world == r]
        seen += out[r]["calls"]
    assert sorted(seen) == list(range(7))
