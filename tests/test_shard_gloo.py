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


def _worker_batched(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2503_22227_b200.pdq.shard import ShardGroup

    g = ShardGroup.from_env()
    batches, singles = [], []

    def fn(u):
        singles.append(u)
        return (torch.arange(4, dtype=torch.int64) * (u + 1), None)

    def batch_fn(us):
        if us[0] % 3 == 2:  # this key's batch declines -> per-unit fallback
            return None
        batches.append(list(us))
        return [(torch.arange(4, dtype=torch.int64) * (u + 1), None) for u in us]

    res = g.map_units_batched(list(range(9)), fn, batch_fn, key=lambda u: u % 3)
    out[rank] = {"batches": batches, "singles": singles,
                 "res": [r[0].tolist() for r in res]}
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [1, 2])
def test_units_batched_per_rank(world):
    """map_units_batched: each rank batches the units it owns by key, falls
    back to per-unit calls when a batch declines, and every rank ends with
    all results."""
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker_batched, args=(world, port, out), nprocs=world, join=True)
    want = [[v * (u + 1) for v in range(4)] for u in range(9)]
    done = []
    for r in range(world):
        assert out[r]["res"] == want
        owned = [u for u in range(9) if u % world == r]
        for b in out[r]["batches"]:
            assert len(b) > 1 and all(u in owned for u in b) and len({u % 3 for u in b}) == 1
        done += [u for b in out[r]["batches"] for u in b] + out[r]["singles"]
    assert sorted(done) == list(range(9))
