"""Multi-process PDQ workers for tests/test_gpu_pdq_shard.py: every rank is a
process on the leased GPU (cuda:0), joined over gloo (which carries the CUDA
tensors through host memory); the production bench runs the same code over
NCCL with one GPU per rank."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def _init(rank, world, port):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)


def session(rows=1024):
    """The reference PdqClient keying (seed 1) at config 5."""
    from paper_2503_22227_b200.context import Context, PoolConfig, Scheme, params_for_profile
    from paper_2503_22227_b200.coremath.sampling import Rng
    from paper_2503_22227_b200.keys import galois_keygen, keygen, pk_gen, relin_keygen
    from paper_2503_22227_b200.pdq.config import PdqConfig
    from paper_2503_22227_b200.pdq.evaluator import CkksEval, rotation_steps

    cfg = PdqConfig(base=4, digits=8, rows=rows, value_bound=1 << 16, profile="pdq")
    ctx = Context(params_for_profile("pdq", Scheme.CKKS), PoolConfig(unit_mb=64, cap_mb=2048))
    rng = Rng((1).to_bytes(32, "little"))
    sk = keygen(ctx, rng)
    pk = pk_gen(ctx, sk, rng)
    rlk = relin_keygen(ctx, sk, rng)
    gks = galois_keygen(ctx, sk, rotation_steps(ctx.n), rng)
    return cfg, ctx, sk, pk, CkksEval(ctx, rlk, gks), rng


def units_worker(rank, world, port, out):
    """Standard queries 1..4 with the (atom, digit) units split over ranks;
    returns the result digests (must equal the reference run's)."""
    import numpy as np
    import torch.distributed as dist

    from fhe_testutil import digest
    from paper_2503_22227_b200.pdq.columns import encode_column
    from paper_2503_22227_b200.pdq.dataset import make_dataset
    from paper_2503_22227_b200.pdq.engine import (LocalInverseClient, PdqEngine,
                                                  encrypt_query_constants, standard_query)
    from paper_2503_22227_b200.pdq.shard import ShardGroup

    _init(rank, world, port)
    cfg, ctx, sk, pk, ev, rng = session()
    group = ShardGroup.from_env()
    engine = PdqEngine(ev, cfg, group=group)
    for name, vals in make_dataset(cfg, seed=20240117).items():
        engine.add_column(encode_column(ev, cfg, name, vals, pk, rng))
    inv = LocalInverseClient(ev, cfg, sk, pk, rng=rng)
    mask_rng = np.random.default_rng(20240118)
    res = {}
    for qid in (1, 2, 3, 4):
        spec = standard_query(qid)
        temps = encrypt_query_constants(ev, cfg, spec, pk, rng)
        r = engine.run(spec, channel=inv, temps=temps, rng=mask_rng)
        res[str(qid)] = {k: [digest(c.data.view()), c.scale, c.level] for k, c in r.cts.items()}
    out[rank] = json.dumps(res)
    dist.barrier()
    dist.destroy_process_group()


def rowblocks_worker(rank, world, port, out, rows=4 * 2048):
    """Row-batch layout: 'sum' and 'avg' aggregates over `rows` rows split in
    blocks of N/2; returns aggregate digests and decrypted values."""
    import numpy as np
    import torch.distributed as dist

    from fhe_testutil import digest
    from paper_2503_22227_b200.pdq.config import PdqConfig  # noqa: F401
    from paper_2503_22227_b200.pdq.dataset import make_dataset
    from paper_2503_22227_b200.pdq.engine import LocalInverseClient, standard_query
    from paper_2503_22227_b200.pdq.rowblocks import RowBlockEngine
    from paper_2503_22227_b200.pdq.shard import ShardGroup

    if world > 1:
        _init(rank, world, port)
        group = ShardGroup.from_env()
    else:
        import torch

        torch.cuda.set_device(0)
        group = ShardGroup(0, 1)
    cfg, ctx, sk, pk, ev, rng = session(rows)
    data = make_dataset(cfg, seed=20240117)
    eng = RowBlockEngine(ev, cfg, group)
    eng.load(data, pk, seed=100)
    inv = LocalInverseClient(ev, cfg, sk, pk, rng=rng)
    res = {"blocks": eng.blocks_of_rank()}
    for qid in (2, 4):
        r = eng.run(standard_query(qid), pk, channel=inv, rng=np.random.default_rng(5))
        res[str(qid)] = {k: digest(c.data.view()) for k, c in r.cts.items() if k != "avg"}
        res[f"{qid}_dec"] = {k: float(ev.decrypt(c, sk).real[0]) for k, c in r.cts.items()}
    out[rank] = json.dumps(res)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
