"""Experiment timer (one GPU): wall time of each step of the PDQ avg query (q4)'s
host part (two-party inverse and the products after it), config 5, after
warm-up.  Not a benchmark."""
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

cfg, ctx, sk, pk, ev, rng = pdq_workers.session()
engine = PdqEngine(ev, cfg)
for name, vals in make_dataset(cfg).items():
    engine.add_column(encode_column(ev, cfg, name, vals, pk, rng))
inv = LocalInverseClient(ev, cfg, sk, pk, rng=rng)
mr = np.random.default_rng(1)
spec = standard_query(4)
parts = engine.device_part(spec, {})
torch.cuda.synchronize()

steps = {}


def t(name, fn):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = fn()
    torch.cuda.synchronize()
    steps.setdefault(name, []).append((time.perf_counter() - t0) * 1e3)
    return r


for _ in range(8):
    ct = parts["count"]
    e = cfg.mask_exp_range
    r = mr.uniform(2.0 ** -e, 2.0 ** e, ev.slots) * mr.choice([-1.0, 1.0], ev.slots)
    masked = t("mul_plain_vec(count, r)", lambda: ev.mul_plain_vec(ct, r))
    vals = t("decrypt", lambda: ev.decrypt(masked, sk).real)
    recip = t("host reciprocal", lambda: np.where(np.abs(vals) < cfg.recip_threshold, 0.0,
                                                 1.0 / np.where(np.abs(vals) < cfg.recip_threshold,
                                                                1.0, vals)))
    scale = ev.ctx.params.default_scale * 2.0 ** 20
    fresh = t("encrypt", lambda: ev.encrypt(recip, pk, rng=rng, scale=scale))
    invc = t("mul_plain_vec(fresh, r)", lambda: ev.mul_plain_vec(fresh, r))
    t("mul(total, inv)", lambda: ev.mul(parts["total"], invc))
    t("whole finish", lambda: engine.finish(spec, parts, inv, mr))
for k, v in steps.items():
    print(f"{k:28s} {statistics.median(v[2:]):7.3f} ms")
