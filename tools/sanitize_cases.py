"""Small invocations of every kernel family for compute-sanitizer
(memcheck / racecheck / synccheck): the persistent fused TMA NTT (>= 8 rows
per residue class at N=2^16), the cluster NTT (FHE_NTT_CLUSTER=1), the
hybrid key switch with its finishing kernels (fhe_hmult_relin at batch 8),
rotate and rescale.  Each case is checked against the public API / the
inverse transform, so a run also proves the results survive the tool."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2503_22227_b200 import _native  # noqa: E402
from paper_2503_22227_b200.context import Context, PoolConfig, hybrid_params  # noqa: E402
from paper_2503_22227_b200.coremath.ntt import DeviceChain  # noqa: E402
from paper_2503_22227_b200.coremath.primes import gen_ntt_prime_chain  # noqa: E402
from paper_2503_22227_b200.coremath.sampling import Rng  # noqa: E402
from paper_2503_22227_b200.keys import (galois_keygen, hmult_relin_into, keygen, pk_gen,  # noqa
                                        relin_keygen)
from paper_2503_22227_b200.schemes import ckks  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "all"
n = 1 << 16
# ks_tc: digits of >= 4 limbs and K >= 4, so ModUp / ModDown run on the tcgen05
# conversion (csrc/bconv_umma.cuh) and the finish on the staged kernel;
# ntt12: the N=2^12 row-per-cluster NTT (plain rows and the rescale
# correction's broadcast input)
KS_SHAPE = {"ks": (6, 2), "ks_tc": (12, 4), "ks_p60": (12, 4)}  # ks_p60: 60-bit P (wide tcgen05)
if which in ("all", "ntt"):
    L, rows = 2, 16
    primes = [m.value for m in gen_ntt_prime_chain(50, n, L)]
    ch = DeviceChain(primes, 16)
    q = torch.tensor(primes, dtype=torch.float64, device="cuda")
    a = (torch.rand((rows, n), dtype=torch.float64, device="cuda") * q.repeat(rows // L)[:, None]
         ).to(torch.int64)
    b = a.clone()
    p0 = _native.ntt_path_counts()
    ch.transform(b, rows, False, limbs=L, offset=0)
    ch.transform(b, rows, True, limbs=L, offset=0)
    torch.cuda.synchronize()
    assert torch.equal(a, b), "NTT round trip"
    print("ntt paths", {k: v - p0[k] for k, v in _native.ntt_path_counts().items() if v != p0[k]})
if which in ("ntt12",):
    from paper_2503_22227_b200.context import params_for_profile, Scheme
    n12 = 1 << 12
    primes = [m.value for m in gen_ntt_prime_chain(45, n12, 13)]
    ch = DeviceChain(primes, 12)
    a = torch.randint(0, 1 << 44, (13, n12), dtype=torch.int64, device="cuda")
    b = a.clone()
    p0 = _native.ntt_path_counts()
    ch.transform(b, 13, False, limbs=13, offset=0)
    ch.transform(b, 13, True, limbs=13, offset=0)
    torch.cuda.synchronize()
    assert torch.equal(a, b), "N=2^12 NTT round trip"
    ctx = Context(params_for_profile("pdq", Scheme.CKKS), PoolConfig(unit_mb=64, cap_mb=512))
    sk = keygen(ctx, Rng((1).to_bytes(32, "little")))
    pk = pk_gen(ctx, sk, Rng((2).to_bytes(32, "little")))
    x = np.random.default_rng(1).uniform(-1, 1, n12 // 2)
    cx = ckks.ckks_encrypt(ctx, ckks.ckks_encode(ctx, x), pk, Rng((3).to_bytes(32, "little")))
    r = ckks.ckks_rescale(ctx, ckks.ckks_multiply_scalar(ctx, cx, 1.0, scale=float(ctx.q_values[-1])))
    torch.cuda.synchronize()
    print("ntt paths", {k: v - p0[k] for k, v in _native.ntt_path_counts().items() if v != p0[k]},
          "rescale level", r.level)
if which in ("all", "ks", "ks_tc", "ks_p60"):
    Lk, Kk = KS_SHAPE.get(which, KS_SHAPE["ks"])
    ctx = Context(hybrid_params(n, Lk, special=Kk, dnum=3, scale=float(2 ** 49),
                                special_bits=60 if which == "ks_p60" else 50),
                  PoolConfig(unit_mb=64, cap_mb=2048))
    seed = lambda s: Rng(int(s).to_bytes(32, "little"))  # noqa: E731
    sk = keygen(ctx, seed(1))
    pk = pk_gen(ctx, sk, seed(2))
    rlk = relin_keygen(ctx, sk, seed(3))
    gks = galois_keygen(ctx, sk, [1], seed(4))
    x = np.random.default_rng(1).uniform(-1, 1, n // 2)
    cx = ckks.ckks_encrypt(ctx, ckks.ckks_encode(ctx, x), pk, seed(5))
    B, Lv = 8, ctx.L
    X = torch.stack([cx.data.view()] * B)
    for i in range(1, B):
        X[i] = ckks.ckks_add(ctx, ckks.CkksCiphertext(ckks.CData.wrap(X[i - 1].reshape(-1), 2, Lv, n,
                                                                       ckks.Domain.EVALUATION),
                                                       cx.scale, Lv), cx).data.view()
    out = torch.empty_like(X)
    hmult_relin_into(ctx, Lv, X, X, rlk, out[:, 0], out[:, 1], batch=B)
    for i in (0, B - 1):
        ct = ckks.CkksCiphertext(ckks.CData.wrap(X[i].reshape(-1), 2, Lv, n, ckks.Domain.EVALUATION),
                                 cx.scale, Lv)
        ref = ckks.ckks_relinearize(ctx, ckks.ckks_multiply(ctx, ct, ct), rlk)
        assert torch.equal(out[i], ref.data.view()), f"hmult_relin item {i}"
        ckks.ckks_rotate(ctx, ct, 1, gks)
        ckks.ckks_rescale(ctx, ref)
    torch.cuda.synchronize()
    print("key switch / rotate / rescale ok")
print("sanitize cases done:", which)
