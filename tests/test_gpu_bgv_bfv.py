"""BGV and BFV (incl. BEHZ) on the B200 vs the reference: bit-identical
ciphertexts at the reference test-suite's n=64 shape and at config 3
(N=2^14, Q = 8 x 50-bit, t = 65537), exact decryption mod t."""

import numpy as np
import pytest

from fhe_testutil import digest, seeded_rng, to_u64

pytestmark = pytest.mark.gpu


def _ctx(scheme, n, moduli):
    from paper_2503_22227_b200.context import Context, EncryptionParams, PoolConfig

    return Context(EncryptionParams(scheme, n, tuple(moduli), plain_modulus=65537),
                   PoolConfig(unit_mb=64, cap_mb=1024))


@pytest.mark.parametrize("tag", ["bgv", "bfv"])
def test_small_pipeline_bit_identical(tag, golden, golden_arrays):
    from paper_2503_22227_b200.context import Scheme
    from paper_2503_22227_b200.coremath.primes import gen_ntt_prime_chain
    from paper_2503_22227_b200.keys import galois_keygen, keygen, pk_gen, relin_keygen
    from paper_2503_22227_b200.schemes import bfv, bgv
    from paper_2503_22227_b200.schemes.batching import batch_decode

    s = golden_arrays["small"]
    mod = bgv if tag == "bgv" else bfv
    ctx = _ctx(Scheme(tag), 64, [m.value for m in gen_ntt_prime_chain(36, 64, 3)])
    sk = keygen(ctx, seeded_rng(1))
    pk = pk_gen(ctx, sk, seeded_rng(2))
    rlk = relin_keygen(ctx, sk, seeded_rng(3))
    gks = galois_keygen(ctx, sk, [1], seeded_rng(4), include_conj=True)
    va, vb = s[f"{tag}_va"], s[f"{tag}_vb"]
    ca = getattr(mod, f"{tag}_encrypt_ints")(ctx, va, pk, seeded_rng(10))
    cb = getattr(mod, f"{tag}_encrypt_ints")(ctx, vb, pk, seeded_rng(11))
    assert (to_u64(ca.data.view()) == s[f"{tag}_ca"]).all()
    assert (to_u64(cb.data.view()) == s[f"{tag}_cb"]).all()
    prod = getattr(mod, f"{tag}_multiply")(ctx, ca, cb)
    assert (to_u64(prod.data.view()) == s[f"{tag}_prod"]).all()
    lin = getattr(mod, f"{tag}_relinearize")(ctx, prod, rlk)
    assert (to_u64(lin.data.view()) == s[f"{tag}_lin"]).all()
    rot = getattr(mod, f"{tag}_rotate_rows")(ctx, ca, 1, gks)
    assert (to_u64(rot.data.view()) == s[f"{tag}_rot"]).all()
    if tag == "bgv":
        ms = bgv.bgv_mod_switch(ctx, lin)
        assert (to_u64(ms.data.view()) == s["bgv_ms"]).all()
        assert ms.plain_factor == golden["small"]["bgv_ms_factor"]
        got = batch_decode(ctx, bgv.bgv_decrypt(ctx, ms, sk))
    else:
        got = batch_decode(ctx, bfv.bfv_decrypt(ctx, lin, sk))
    assert (got == s[f"{tag}_dec"]).all()
    assert got.tolist() == (va.astype(object) * vb % 65537).tolist()


@pytest.mark.parametrize("tag", ["bgv", "bfv"])
def test_config3_bit_identical_and_exact(tag, golden):
    from paper_2503_22227_b200.context import Scheme
    from paper_2503_22227_b200.keys import keygen, pk_gen, relin_keygen
    from paper_2503_22227_b200.schemes import bfv, bgv
    from paper_2503_22227_b200.schemes.batching import batch_decode

    g = golden["c3"]
    mod = bgv if tag == "bgv" else bfv
    n = 1 << 14
    ctx = _ctx(Scheme(tag), n, [int(q) for q in g["primes"]])
    sk = keygen(ctx, seeded_rng(3))
    pk = pk_gen(ctx, sk, seeded_rng(31))
    rlk = relin_keygen(ctx, sk, seeded_rng(32))
    vr = np.random.default_rng(5)
    va = vr.integers(0, 65537, n, dtype=np.uint64)
    vb = vr.integers(0, 65537, n, dtype=np.uint64)
    ca = getattr(mod, f"{tag}_encrypt_ints")(ctx, va, pk, seeded_rng(33))
    cb = getattr(mod, f"{tag}_encrypt_ints")(ctx, vb, pk, seeded_rng(34))
    assert digest(ca.data.view()) == g[tag]["ca"]
    assert digest(cb.data.view()) == g[tag]["cb"]
    prod = getattr(mod, f"{tag}_multiply")(ctx, ca, cb)
    assert digest(prod.data.view()) == g[tag]["prod"]
    lin = getattr(mod, f"{tag}_relinearize")(ctx, prod, rlk)
    assert digest(lin.data.view()) == g[tag]["lin"]
    dec = (bgv.bgv_decrypt if tag == "bgv" else bfv.bfv_decrypt)(ctx, lin, sk)
    assert batch_decode(ctx, dec).tolist() == (va.astype(object) * vb % 65537).tolist()
