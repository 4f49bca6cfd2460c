"""Generate golden vectors by running the REFERENCE implementation.

Run in the build container only (needs /root/reference; the GPU box does
not have it):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_golden.py [--big]

Every input is derived from a seed, so the fixtures store small arrays in
full and large ones as SHA-256 digests of their little-endian uint64 bytes;
the GPU tests regenerate the same inputs from the same seeds.
Outputs: tests/golden/ntt.npz, ckks_c1.npz, small.npz, digests.json
(and ckks_c4.json with --big: N=2^16, L=30, reference gadget).
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

import rnsfhe.context as rctx  # noqa: E402
from rnsfhe.context import Context, EncryptionParams, Scheme, params_for_profile  # noqa: E402
from rnsfhe.coremath.ntt import NttChain, NttTables  # noqa: E402
from rnsfhe.coremath.primes import gen_ntt_prime_chain  # noqa: E402
from rnsfhe.coremath.sampling import Rng  # noqa: E402
from rnsfhe.keys import galois_keygen, key_switch, keygen, pk_gen, relin_keygen  # noqa: E402
from rnsfhe.schemes import bfv, bgv, ckks  # noqa: E402
from rnsfhe.schemes.batching import batch_decode  # noqa: E402


def digest(a) -> str:
    a = np.ascontiguousarray(np.asarray(a, dtype=np.uint64))
    return hashlib.sha256(a.astype("<u8").tobytes()).hexdigest()


def seeded(seed: int) -> Rng:
    return Rng(int(seed).to_bytes(32, "little"))


def ntt_inputs(primes, n, rows, seed):
    """Config-2 style input: row r uniform mod q_{r % L}."""
    rng = np.random.default_rng(seed)
    L = len(primes)
    return np.stack([rng.integers(0, primes[r % L], n, dtype=np.uint64) for r in range(rows)])


# NTT cases: (log_n, L, rows, bits, seed); full arrays for small, digests for big
NTT_CASES = [
    (2, 2, 4, 36, 1), (4, 2, 4, 36, 2), (6, 3, 6, 36, 3), (8, 3, 6, 45, 4), (10, 2, 4, 50, 5),
    (12, 4, 8, 50, 6), (13, 3, 6, 45, 7), (14, 2, 2, 50, 8), (15, 2, 2, 50, 9),
    (16, 3, 3, 50, 10), (17, 1, 1, 50, 11), (12, 40, 80, 50, 20261017), (16, 30, 30, 50, 12),
]
FULL_LIMIT = 1 << 14  # words stored in full below this


def gen_ntt(out):
    arrays, meta = {}, []
    for log_n, L, rows, bits, seed in NTT_CASES:
        n = 1 << log_n
        primes = [m.value for m in gen_ntt_prime_chain(bits, n, L)]
        chain = NttChain([NttTables(n, m) for m in gen_ntt_prime_chain(bits, n, L)])
        a = ntt_inputs(primes, n, rows, seed)
        midx = np.arange(rows) % L
        fwd = chain.forward(a, midx)
        inv = chain.inverse(a, midx)
        key = f"n{log_n}_L{L}_r{rows}_b{bits}"
        rec = {"key": key, "log_n": log_n, "L": L, "rows": rows, "bits": bits, "seed": seed,
               "primes": [str(p) for p in primes],
               "psi": [str(t.psi) for t in chain.tables],
               "fwd_sha": digest(fwd), "inv_sha": digest(inv), "in_sha": digest(a)}
        if rows * n <= FULL_LIMIT:
            arrays[key + "_in"] = a
            arrays[key + "_fwd"] = fwd
            arrays[key + "_inv"] = inv
        # the first 64 twiddles of prime 0, both directions (table pinning)
        arrays[key + "_psi_br"] = chain.tables[0].psi_powers[:64]
        arrays[key + "_ipsi_br"] = chain.tables[0].inv_psi_powers[:64]
        meta.append(rec)
    np.savez_compressed(os.path.join(HERE, "ntt.npz"), **arrays)
    out["ntt"] = meta


def ct_digest(ct):
    return digest(ct.data.view())


def gen_ckks_c1(out):
    """Config 1: CKKS N=2^13, 3 x 45-bit, Delta = 2^44."""
    n = 8192
    moduli = tuple(m.value for m in gen_ntt_prime_chain(45, n, 3))
    p = EncryptionParams(Scheme.CKKS, n, moduli, default_scale=float(2 ** 44))
    ctx = Context(p)
    sk = keygen(ctx, seeded(1))
    pk = pk_gen(ctx, sk, seeded(2))
    rlk = relin_keygen(ctx, sk, seeded(3))
    gks = galois_keygen(ctx, sk, [1, 5], seeded(4), include_conj=True)
    vr = np.random.default_rng(1)
    x = vr.uniform(-1, 1, n // 2)
    y = vr.uniform(-1, 1, n // 2)
    ptx = ckks.ckks_encode(ctx, x)
    cx = ckks.ckks_encrypt(ctx, ptx, pk, seeded(10))
    cy = ckks.ckks_encrypt(ctx, ckks.ckks_encode(ctx, y), pk, seeded(11))
    prod = ckks.ckks_multiply(ctx, cx, cy)
    sq = ckks.ckks_square(ctx, cx)
    lin = ckks.ckks_relinearize(ctx, prod, rlk)
    res = ckks.ckks_rescale(ctx, lin)
    rot = ckks.ckks_rotate(ctx, cx, 1, gks)
    rot5 = ckks.ckks_rotate(ctx, cx, 5, gks)
    conj = ckks.ckks_conjugate(ctx, cx, gks)
    dec = ckks.ckks_decode(ctx, ckks.ckks_decrypt(ctx, res, sk))
    dec_x = ckks.ckks_decode(ctx, ckks.ckks_decrypt(ctx, cx, sk))
    boosted = ckks.ckks_rescale(ctx, ckks.ckks_rotate(
        ctx, ckks.ckks_multiply_scalar(ctx, cx, 1.0, scale=float(moduli[-1])), 1, gks))
    dec_rot = ckks.ckks_decode(ctx, ckks.ckks_decrypt(ctx, boosted, sk))
    ks_b, ks_a = key_switch(ctx, cy.data.view()[1], rlk)
    rec = {
        "n": n, "primes": [str(q) for q in moduli], "scale": 2.0 ** 44,
        "sk_s": digest(sk.s.view()), "pk": digest(pk.data.view()),
        "rlk": [digest(d.view()) for d in rlk.digits],
        "gk": {str(e): [digest(d.view()) for d in k.digits] for e, k in gks.keys.items()},
        "pt_x": digest(ptx.data.view()),
        "ct_x": ct_digest(cx), "ct_y": ct_digest(cy), "prod": ct_digest(prod),
        "square": ct_digest(sq), "relin": ct_digest(lin), "rescale": ct_digest(res),
        "rescale_scale": res.scale, "rot1": ct_digest(rot), "rot5": ct_digest(rot5),
        "conj": ct_digest(conj), "boosted_rot": ct_digest(boosted),
        "ks_b": digest(ks_b), "ks_a": digest(ks_a),
        "err_mul": float(np.max(np.abs(dec - x * y))),
        "err_enc": float(np.max(np.abs(dec_x - x))),
        "err_rot": float(np.max(np.abs(dec_rot - np.roll(x, -1)))),
    }
    np.savez_compressed(os.path.join(HERE, "ckks_c1.npz"), dec_mul=dec, dec_x=dec_x,
                        dec_rot=dec_rot, sk_coeffs=sk.coeffs)
    out["ckks_c1"] = rec


def small_ctx(scheme, n=64, levels=3, bits=36):
    moduli = tuple(m.value for m in gen_ntt_prime_chain(bits, n, levels))
    if scheme is Scheme.CKKS:
        return Context(EncryptionParams(scheme, n, moduli, default_scale=float(1 << (bits - 1))))
    return Context(EncryptionParams(scheme, n, moduli, plain_modulus=65537))


def gen_small(out):
    """n = 64 contexts (the reference test-suite's shapes): full arrays."""
    arrays = {}
    rec = {}
    # CKKS small: key switch full arrays
    ctx = small_ctx(Scheme.CKKS)
    sk = keygen(ctx, seeded(5))
    rk = relin_keygen(ctx, sk, seeded(9))
    d = ctx.ntt_chain.forward(seeded(11).uniform_residues(ctx.q_arr(), ctx.n), np.arange(3))
    b, a = key_switch(ctx, d, rk)
    arrays.update(ks_sk=sk.s.view(), ks_d=d, ks_b=b, ks_a=a,
                  ks_rlk=np.stack([x.view() for x in rk.digits]))
    # BGV at n = 64 (t = 65537): encrypt, multiply, relin, mod switch, rotate
    for scheme, mod in ((Scheme.BGV, bgv), (Scheme.BFV, bfv)):
        ctx = small_ctx(scheme)
        tag = scheme.value
        sk = keygen(ctx, seeded(1))
        pk = pk_gen(ctx, sk, seeded(2))
        rlk = relin_keygen(ctx, sk, seeded(3))
        gks = galois_keygen(ctx, sk, [1], seeded(4), include_conj=True)
        vr = np.random.default_rng(7)
        va = vr.integers(0, 65537, 64, dtype=np.uint64)
        vb = vr.integers(0, 65537, 64, dtype=np.uint64)
        ca = getattr(mod, f"{tag}_encrypt_ints")(ctx, va, pk, seeded(10))
        cb = getattr(mod, f"{tag}_encrypt_ints")(ctx, vb, pk, seeded(11))
        prod = getattr(mod, f"{tag}_multiply")(ctx, ca, cb)
        lin = getattr(mod, f"{tag}_relinearize")(ctx, prod, rlk)
        rot = getattr(mod, f"{tag}_rotate_rows")(ctx, ca, 1, gks)
        arrays.update({f"{tag}_ca": ca.data.view(), f"{tag}_cb": cb.data.view(),
                       f"{tag}_prod": prod.data.view(), f"{tag}_lin": lin.data.view(),
                       f"{tag}_rot": rot.data.view(), f"{tag}_va": va, f"{tag}_vb": vb})
        if scheme is Scheme.BGV:
            ms = bgv.bgv_mod_switch(ctx, lin)
            arrays[f"{tag}_ms"] = ms.data.view()
            rec["bgv_ms_factor"] = int(ms.plain_factor)
            got = batch_decode(ctx, bgv.bgv_decrypt(ctx, ms, sk))
        else:
            got = batch_decode(ctx, bfv.bfv_decrypt(ctx, lin, sk))
        arrays[f"{tag}_dec"] = got
    np.savez_compressed(os.path.join(HERE, "small.npz"), **arrays)
    out["small"] = rec


def gen_bgv_c3(out):
    """Config 3: BFV and BGV, N = 2^14, Q = 8 x 50-bit, t = 65537 (digests)."""
    n = 1 << 14
    moduli = tuple(m.value for m in gen_ntt_prime_chain(50, n, 8))
    rec = {"primes": [str(q) for q in moduli]}
    for scheme, mod in ((Scheme.BGV, bgv), (Scheme.BFV, bfv)):
        tag = scheme.value
        ctx = Context(EncryptionParams(scheme, n, moduli, plain_modulus=65537))
        sk = keygen(ctx, seeded(3))
        pk = pk_gen(ctx, sk, seeded(31))
        rlk = relin_keygen(ctx, sk, seeded(32))
        vr = np.random.default_rng(5)
        va = vr.integers(0, 65537, n, dtype=np.uint64)
        vb = vr.integers(0, 65537, n, dtype=np.uint64)
        t0 = time.perf_counter()
        ca = getattr(mod, f"{tag}_encrypt_ints")(ctx, va, pk, seeded(33))
        cb = getattr(mod, f"{tag}_encrypt_ints")(ctx, vb, pk, seeded(34))
        prod = getattr(mod, f"{tag}_multiply")(ctx, ca, cb)
        lin = getattr(mod, f"{tag}_relinearize")(ctx, prod, rlk)
        rec[tag] = {"ca": ct_digest(ca), "cb": ct_digest(cb), "prod": ct_digest(prod),
                    "lin": ct_digest(lin), "seconds": time.perf_counter() - t0}
        dec = (bgv.bgv_decrypt if scheme is Scheme.BGV else bfv.bfv_decrypt)(ctx, lin, sk)
        got = batch_decode(ctx, dec)
        want = (va.astype(object) * vb % 65537).astype(np.uint64)
        rec[tag]["exact"] = bool((got == want).all())
    out["c3"] = rec


def gen_ckks_c4(out):
    """Config 4 in the reference gadget (alpha=1, K=0): N=2^16, L=30."""
    rctx.MAX_CHAIN_LEN = 30
    n = 1 << 16
    moduli = tuple(m.value for m in gen_ntt_prime_chain(50, n, 30))
    ctx = Context(EncryptionParams(Scheme.CKKS, n, moduli, default_scale=float(2 ** 49)))
    sk = keygen(ctx, seeded(4))
    pk = pk_gen(ctx, sk, seeded(41))
    t0 = time.perf_counter()
    rlk = relin_keygen(ctx, sk, seeded(42))
    t_key = time.perf_counter() - t0
    vr = np.random.default_rng(9)
    x = vr.uniform(-1, 1, n // 2)
    y = vr.uniform(-1, 1, n // 2)
    cx = ckks.ckks_encrypt(ctx, ckks.ckks_encode(ctx, x), pk, seeded(43))
    cy = ckks.ckks_encrypt(ctx, ckks.ckks_encode(ctx, y), pk, seeded(44))
    t0 = time.perf_counter()
    prod = ckks.ckks_multiply(ctx, cx, cy)
    t_mul = time.perf_counter() - t0
    t0 = time.perf_counter()
    lin = ckks.ckks_relinearize(ctx, prod, rlk)
    t_relin = time.perf_counter() - t0
    t0 = time.perf_counter()
    res = ckks.ckks_rescale(ctx, lin)
    t_rs = time.perf_counter() - t0
    dec = ckks.ckks_decode(ctx, ckks.ckks_decrypt(ctx, res, sk))
    out["ckks_c4"] = {
        "primes": [str(q) for q in moduli], "scale": 2.0 ** 49,
        "sk_s": digest(sk.s.view()), "rlk0": digest(rlk.digits[0].view()),
        "rlk29": digest(rlk.digits[29].view()),
        "ct_x": ct_digest(cx), "ct_y": ct_digest(cy), "prod": ct_digest(prod),
        "relin": ct_digest(lin), "rescale": ct_digest(res),
        "err_mul": float(np.max(np.abs(dec - x * y))),
        "seconds": {"relin_keygen": t_key, "multiply": t_mul, "relinearize": t_relin,
                    "rescale": t_rs},
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--big", action="store_true", help="also run config 3 and config 4")
    ap.add_argument("--pdq", action="store_true", help="(separate entry) config 5 queries")
    args = ap.parse_args()
    path = os.path.join(HERE, "digests.json")
    out = json.load(open(path)) if os.path.exists(path) else {}
    out["numpy"] = np.__version__
    gen_ntt(out)
    gen_ckks_c1(out)
    gen_small(out)
    if args.big:
        gen_bgv_c3(out)
        gen_ckks_c4(out)
    json.dump(out, open(path, "w"), indent=1, sort_keys=True)
    print("wrote", path)


if __name__ == "__main__" and "--pdq" not in sys.argv:
    main()


def gen_pdq(out):
    """Config 5: the four standard queries over 1024 synthetic rows, keyed and
    seeded exactly like the reference PdqClient (client seed 1, one Rng for
    keys, columns and the reciprocal replies; server mask seed 20240118)."""
    from rnsfhe.coremath.sampling import Rng as RRng
    from rnsfhe.pdq.columns import encode_column
    from rnsfhe.pdq.config import PdqConfig
    from rnsfhe.pdq.dataset import make_dataset, oracle_result
    from rnsfhe.pdq.engine import (LocalInverseClient, PdqEngine, encrypt_query_constants,
                                   interpret_result, standard_query)
    from rnsfhe.pdq.evaluator import CkksEval, rotation_steps

    cfg = PdqConfig(base=4, digits=8, rows=1024, value_bound=1 << 16, profile="pdq")
    ctx = Context(params_for_profile("pdq", Scheme.CKKS))
    rng = RRng((1).to_bytes(32, "little"))
    sk = keygen(ctx, rng)
    pk = pk_gen(ctx, sk, rng)
    rlk = relin_keygen(ctx, sk, rng)
    gks = galois_keygen(ctx, sk, rotation_steps(ctx.n), rng)
    ev = CkksEval(ctx, rlk, gks)
    data = make_dataset(cfg, seed=20240117)
    engine = PdqEngine(ev, cfg)
    col_digests = {}
    for name, vals in data.items():
        col = encode_column(ev, cfg, name, vals, pk, rng)
        engine.add_column(col)
        col_digests[name] = [digest(c.data.view()) for c in col.digits] + [digest(col.value.data.view())]
    inverse = LocalInverseClient(ev, cfg, sk, pk, rng=rng)
    mask_rng = np.random.default_rng(20240118)
    res = {}
    for qid in (1, 2, 3, 4):
        spec = standard_query(qid)
        temps = encrypt_query_constants(ev, cfg, spec, pk, rng)
        t0 = time.perf_counter()
        result = engine.run(spec, channel=inverse, temps=temps, rng=mask_rng)
        secs = time.perf_counter() - t0
        got = interpret_result(ev, sk, result, cfg.rows)
        want = oracle_result(spec, data)
        rec = {"seconds": secs,
               "cts": {k: {"sha": digest(c.data.view()), "scale": c.scale, "level": c.level}
                       for k, c in result.cts.items()}}
        if spec.agg == "index":
            rec["value"] = np.asarray(got).astype(int).tolist()
            rec["oracle_match"] = bool((np.asarray(got) == want).all())
        elif spec.agg == "ratio":
            rec["value_sha"] = hashlib.sha256(np.asarray(got, dtype=np.float64).tobytes()).hexdigest()
            rec["max_err"] = float(np.max(np.abs(np.asarray(got) - want)))
        else:
            rec["value"] = got if not isinstance(got, tuple) else list(got)
            rec["oracle"] = want if not isinstance(want, tuple) else list(want)
        res[str(qid)] = rec
    out["pdq"] = {"columns": col_digests, "queries": res, "n": ctx.n,
                  "primes": [str(q) for q in ctx.q_values]}


if __name__ == "__main__" and "--pdq" in sys.argv:
    path = os.path.join(HERE, "digests.json")
    o = json.load(open(path))
    gen_pdq(o)
    json.dump(o, open(path, "w"), indent=1, sort_keys=True)
    print("wrote pdq goldens")
