"""PDQ query profile helper (run under ncu or plain): builds the config-5
engine, runs one warm query, then one query inside an NVTX range "pdq".

    python tools/pdq_profile.py [query_id]
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402


def main(qid=1):
    from paper_2503_22227_b200.context import Context, PoolConfig, Scheme, params_for_profile
    from paper_2503_22227_b200.coremath.sampling import Rng
    from paper_2503_22227_b200.keys import galois_keygen, keygen, pk_gen, relin_keygen
    from paper_2503_22227_b200.pdq.columns import encode_column
    from paper_2503_22227_b200.pdq.config import PdqConfig
    from paper_2503_22227_b200.pdq.dataset import make_dataset
    from paper_2503_22227_b200.pdq.engine import LocalInverseClient, PdqEngine, standard_query
    from paper_2503_22227_b200.pdq.evaluator import CkksEval, rotation_steps

    cfg = PdqConfig()
    ctx = Context(params_for_profile("pdq", Scheme.CKKS), PoolConfig(unit_mb=64, cap_mb=2048))
    rng = Rng((1).to_bytes(32, "little"))
    sk = keygen(ctx, rng)
    pk = pk_gen(ctx, sk, rng)
    ev = CkksEval(ctx, relin_keygen(ctx, sk, rng),
                  galois_keygen(ctx, sk, rotation_steps(ctx.n), rng))
    engine = PdqEngine(ev, cfg)
    for name, vals in make_dataset(cfg).items():
        engine.add_column(encode_column(ev, cfg, name, vals, pk, rng))
    inv = LocalInverseClient(ev, cfg, sk, pk, rng=rng)
    mask_rng = np.random.default_rng(20240118)
    spec = standard_query(qid)
    engine.run(spec, channel=inv, rng=mask_rng)
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_push("pdq")
    t0 = time.perf_counter()
    engine.run(spec, channel=inv, rng=mask_rng)
    torch.cuda.synchronize()
    print(f"query {qid}: {1e3 * (time.perf_counter() - t0):.1f} ms wall")
    torch.cuda.nvtx.range_pop()


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 1)
