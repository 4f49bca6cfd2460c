"""Run in a subprocess with FHE_NTT_CLUSTER=1 (the path switch is read once
per process): the one-pass cluster NTT at N=2^16 vs the C oracle for
several row counts (odd, fewer rows than clusters, batch-strided classes).
Prints one JSON line."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import fast  # noqa: E402
from paper_2503_22227_b200 import _native  # noqa: E402
from paper_2503_22227_b200.coremath.ntt import DeviceChain  # noqa: E402
from paper_2503_22227_b200.coremath.primes import gen_ntt_prime_chain  # noqa: E402

n = 1 << 16
out = {}
for L, rows in ((3, 7), (5, 640), (30, 90)):
    primes = [m.value for m in gen_ntt_prime_chain(50, n, L)]
    rng = np.random.default_rng(rows)
    q = np.array(primes, dtype=np.uint64)[np.arange(rows) % L]
    a = (rng.integers(0, 1 << 62, (rows, n), dtype=np.uint64) % q[:, None]).astype(np.uint64)
    ch = DeviceChain(primes, 16)
    midx = np.arange(rows) % L
    for inverse in (False, True):
        buf = torch.from_numpy(a.view(np.int64)).cuda()
        c0 = _native.ntt_path_counts()["cluster"]
        ch.transform(buf, rows, inverse, limbs=L, offset=0)
        torch.cuda.synchronize()
        took = _native.ntt_path_counts()["cluster"] - c0
        want = fast.ntt_forward(a, primes, midx, inverse=inverse)
        got = buf.cpu().numpy().view(np.uint64)
        out[f"L{L}_rows{rows}_{'inv' if inverse else 'fwd'}"] = {
            "cluster_launches": int(took), "bad_rows": int((got != want).any(axis=1).sum())}
print(json.dumps(out))
