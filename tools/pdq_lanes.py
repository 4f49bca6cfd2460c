"""PDQ latency: eager vs CUDA-graph replay, with and without the stream
lanes for the unit groups (config 5, 1024 rows)."""
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests", "helpers"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import pdq_workers  # noqa: E402
from paper_2503_22227_b200.pdq.columns import encode_column  # noqa: E402
from paper_2503_22227_b200.pdq.dataset import make_dataset  # noqa: E402
from paper_2503_22227_b200.pdq.engine import LocalInverseClient, PdqEngine, standard_query  # noqa
from paper_2503_22227_b200.pdq.graphs import CapturedQuery  # noqa: E402

cfg, ctx, sk, pk, ev, rng = pdq_workers.session()
engine = PdqEngine(ev, cfg)
for name, vals in make_dataset(cfg).items():
    engine.add_column(encode_column(ev, cfg, name, vals, pk, rng))
inv = LocalInverseClient(ev, cfg, sk, pk, rng=rng)
mr = np.random.default_rng(1)


def med(fn, reps=7):
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append((time.perf_counter() - t0) * 1e3)
    return statistics.median(ts[1:])


out = {}
for q in (1, 2, 3, 4):
    spec = standard_query(q)
    for lanes in (False, True):
        engine.use_lanes = lanes
        out[f"q{q}_eager_lanes{int(lanes)}"] = med(lambda: engine.run(spec, channel=inv, rng=mr))
    engine.use_lanes = False
    for lanes in (False, True):
        cq = CapturedQuery(engine, spec, lanes=lanes)
        out[f"q{q}_graph_lanes{int(lanes)}"] = med(lambda: cq.run(channel=inv, rng=mr))
        out[f"q{q}_replay_only_lanes{int(lanes)}"] = med(lambda: cq.replay())
        del cq
print(json.dumps(out))
