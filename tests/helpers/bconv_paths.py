"""Run with FHE_BCONV_IMMA=0 or 1 / FHE_BCONV_UMMA=0 or 1 (read once per
process): HMult+Relin and rotate at a hybrid N=2^16 parameter set (default
L=17 with a ragged last digit; BCONV_SHAPE=L,special,dnum), batch 3,
printing sha256 digests of the results, so the tcgen05, mma.sync and
FP64-pipe base conversions can be compared word for word."""
import hashlib
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2503_22227_b200.context import Context, PoolConfig, hybrid_params  # noqa: E402
from paper_2503_22227_b200.coremath.sampling import Rng  # noqa: E402
from paper_2503_22227_b200.keys import (galois_keygen, hmult_relin_into, keygen, pk_gen,  # noqa
                                        relin_keygen)
from paper_2503_22227_b200.schemes import ckks  # noqa: E402

n = 1 << 16
# BCONV_SHAPE=L,special,dnum (default 17,6,3: digits of 6/6/5 limbs, K-steps 2)
Lq, Ksp, Dn = (int(v) for v in os.environ.get("BCONV_SHAPE", "17,6,3").split(","))
ctx = Context(hybrid_params(n, Lq, special=Ksp, dnum=Dn, scale=float(2 ** 49)),
              PoolConfig(unit_mb=64, cap_mb=4096))
seed = lambda s: Rng(int(s).to_bytes(32, "little"))  # noqa: E731
sk = keygen(ctx, seed(1))
pk = pk_gen(ctx, sk, seed(2))
rlk = relin_keygen(ctx, sk, seed(3))
gks = galois_keygen(ctx, sk, [3], seed(4))
vr = np.random.default_rng(5)
cts = [ckks.ckks_encrypt(ctx, ckks.ckks_encode(ctx, vr.uniform(-1, 1, n // 2)), pk, seed(10 + i))
       for i in range(3)]
X = torch.stack([c.data.view() for c in cts])
Y = torch.stack([cts[(i + 1) % 3].data.view() for i in range(3)])
out = torch.empty_like(X)
hmult_relin_into(ctx, ctx.L, X, Y, rlk, out[:, 0], out[:, 1], batch=3)
rot = ckks.ckks_rotate(ctx, cts[0], 3, gks)
h = lambda t: hashlib.sha256(t.cpu().numpy().tobytes()).hexdigest()  # noqa: E731
print(json.dumps({"hmult": h(out), "rotate": h(rot.data.view()),
                  "imma": os.environ.get("FHE_BCONV_IMMA", "1")}))
