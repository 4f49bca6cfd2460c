import time, sys
sys.path.insert(0, ".")
import numpy as np, torch
from paper_2503_22227_b200.context import Context, PoolConfig, Scheme, params_for_profile
from paper_2503_22227_b200.coremath.sampling import Rng
from paper_2503_22227_b200.keys import keygen, pk_gen, relin_keygen
from paper_2503_22227_b200.schemes import ckks
ctx = Context(params_for_profile("pdq", Scheme.CKKS), PoolConfig(unit_mb=64, cap_mb=2048))
rng = Rng((1).to_bytes(32, "little"))
sk = keygen(ctx, rng); pk = pk_gen(ctx, sk, rng); rlk = relin_keygen(ctx, sk, rng)
x = ckks.ckks_encrypt(ctx, ckks.ckks_encode(ctx, np.ones(ctx.n // 2)), pk, rng)
def t(name, f, k=300):
    for _ in range(20): f()
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(k): f()
    h = time.perf_counter() - t0
    torch.cuda.synchronize(); w = time.perf_counter() - t0
    print(f"{name:28s} host {1e6*h/k:7.1f} us/call  wall {1e6*w/k:7.1f} us/call")
t("ckks_add", lambda: ckks.ckks_add(ctx, x, x))
t("ckks_rescale", lambda: ckks.ckks_rescale(ctx, x))
t("ckks_multiply", lambda: ckks.ckks_multiply(ctx, x, x))
m = ckks.ckks_multiply(ctx, x, x)
t("ckks_relinearize", lambda: ckks.ckks_relinearize(ctx, m, rlk))
t("ckks_multiply_scalar", lambda: ckks.ckks_multiply_scalar(ctx, x, 0.5))
import cProfile, pstats
pr = cProfile.Profile(); pr.enable()
for _ in range(200): ckks.ckks_rescale(ctx, x)
pr.disable(); torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("tottime").print_stats(12)
