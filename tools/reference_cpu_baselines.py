"""Time the REFERENCE package itself (pure Python + numba, /root/reference) on
this container's host cores, for the CPU baselines the GPU box cannot run
(the reference does not travel there).  Writes
profiles/r2_reference_cpu_baselines.json, which bench.py reports verbatim
beside its own numbers, labelled with where it ran.

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tools/reference_cpu_baselines.py

Measured: PDQ queries 1..4 over 1024 rows (bench.run_pdq, second execution
= warm cal_ms); config-3 BFV and BGV multiply + relinearize at
N=2^14, 8 x 50-bit, t=65537 (median of 3 after a warm-up); the config-2
NTT at N=2^16, L=40, 640 rows (NttChain.forward / inverse).
"""
import json
import os
import platform
import statistics
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor()


def med(fn, reps=3):
    fn()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return statistics.median(ts)


def pdq():
    from rnsfhe.bench import run_pdq

    out = {}
    for q in (1, 2, 3, 4):
        r = run_pdq(q)
        out[f"q{q}_ms"] = r["cal_ms"]
        out[f"q{q}_first_ms"] = r["first_cal_ms"]
    return out


def bfv_bgv():
    from rnsfhe.context import Context, EncryptionParams, Scheme
    from rnsfhe.coremath.primes import gen_ntt_prime_chain
    from rnsfhe.coremath.sampling import Rng
    from rnsfhe.keys import keygen, pk_gen, relin_keygen
    from rnsfhe.schemes import bfv, bgv

    n = 1 << 14
    primes = tuple(m.value for m in gen_ntt_prime_chain(50, n, 8))
    out = {}
    for name, scheme, mod in (("bgv", Scheme.BGV, bgv), ("bfv", Scheme.BFV, bfv)):
        ctx = Context(EncryptionParams(scheme, n, primes, plain_modulus=65537))
        rng = Rng((3).to_bytes(32, "little"))
        sk = keygen(ctx, rng)
        pk = pk_gen(ctx, sk, rng)
        rlk = relin_keygen(ctx, sk, rng)
        vals = np.random.default_rng(5).integers(0, 65537, n)
        enc = getattr(mod, f"{name}_encrypt_ints")
        a = enc(ctx, vals, pk, rng)
        b = enc(ctx, vals, pk, rng)
        mul = getattr(mod, f"{name}_multiply")
        rel = getattr(mod, f"{name}_relinearize")
        out[f"{name}_mul_relin_s"] = med(lambda: rel(ctx, mul(ctx, a, b), rlk))
    return out


def ntt():
    from rnsfhe.coremath.ntt import NttChain, NttTables
    from rnsfhe.coremath.primes import gen_ntt_prime_chain

    n, L = 1 << 16, 40
    mods = gen_ntt_prime_chain(50, n, L)
    primes = [m.value for m in mods]
    rows = 640
    rng = np.random.default_rng(20261017)
    a = np.stack([rng.integers(0, primes[r % L], n, dtype=np.uint64) for r in range(rows)])
    ch = NttChain([NttTables(n, m) for m in mods])
    midx = np.arange(rows) % L
    fwd = med(lambda: ch.forward(a, midx), reps=2)
    inv = med(lambda: ch.inverse(a, midx), reps=2)
    algo = 2.0 * rows * n * 8
    return {"rows": rows, "forward_s": fwd, "inverse_s": inv,
            "forward_gbs": algo / fwd / 1e9, "inverse_gbs": algo / inv / 1e9}


def main():
    import numba

    res = {"where": "build container (no GPU), reference package /root/reference/pkg/src",
           "cpu_model": cpu_model(), "cores": os.cpu_count(),
           "numba_threads": numba.config.NUMBA_NUM_THREADS,
           "numpy": np.__version__, "numba": numba.__version__}
    for name, fn in (("ntt_config2", ntt), ("config3", bfv_bgv), ("pdq_1024_rows", pdq)):
        t0 = time.perf_counter()
        res[name] = fn()
        res[name]["wall_s"] = time.perf_counter() - t0
        print(name, res[name], flush=True)
    with open(os.path.join(ROOT, "profiles", "r2_reference_cpu_baselines.json"), "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
