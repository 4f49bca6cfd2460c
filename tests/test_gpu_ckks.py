"""CKKS on the B200 vs the reference, config 1 (N=2^13, 3 x 45-bit, Delta =
2^44) and the reference test-suite's n=64 shapes: every key, ciphertext and
key-switch output word must be bit-identical to the reference's
(tests/golden/make_golden.py), decrypted slots identical floats."""

import numpy as np
import pytest

from fhe_testutil import digest, seeded_rng, to_u64

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def c1(golden):
    from paper_2503_22227_b200.context import Context, EncryptionParams, Scheme
    from paper_2503_22227_b200.keys import galois_keygen, keygen, pk_gen, relin_keygen

    g = golden["ckks_c1"]
    primes = tuple(int(p) for p in g["primes"])
    ctx = Context(EncryptionParams(Scheme.CKKS, g["n"], primes, default_scale=g["scale"]))
    sk = keygen(ctx, seeded_rng(1))
    return {
        "g": g, "ctx": ctx, "sk": sk,
        "pk": pk_gen(ctx, sk, seeded_rng(2)),
        "rlk": relin_keygen(ctx, sk, seeded_rng(3)),
        "gks": galois_keygen(ctx, sk, [1, 5], seeded_rng(4), include_conj=True),
    }


def test_keys_bit_identical(c1):
    g = c1["g"]
    assert digest(c1["sk"].s.view()) == g["sk_s"]
    assert digest(c1["pk"].data.view()) == g["pk"]
    assert [digest(d.view()) for d in c1["rlk"].digits] == g["rlk"]
    for elt, k in c1["gks"].keys.items():
        assert [digest(d.view()) for d in k.digits] == g["gk"][str(elt)]


def test_pipeline_bit_identical(c1, golden_arrays):
    from paper_2503_22227_b200.keys import key_switch
    from paper_2503_22227_b200.schemes import ckks

    g, ctx, sk = c1["g"], c1["ctx"], c1["sk"]
    n = ctx.n
    vr = np.random.default_rng(1)
    x = vr.uniform(-1, 1, n // 2)
    y = vr.uniform(-1, 1, n // 2)
    ptx = ckks.ckks_encode(ctx, x)
    assert digest(ptx.data.view()) == g["pt_x"]
    cx = ckks.ckks_encrypt(ctx, ptx, c1["pk"], seeded_rng(10))
    cy = ckks.ckks_encrypt(ctx, ckks.ckks_encode(ctx, y), c1["pk"], seeded_rng(11))
    assert digest(cx.data.view()) == g["ct_x"]
    assert digest(cy.data.view()) == g["ct_y"]
    prod = ckks.ckks_multiply(ctx, cx, cy)
    assert digest(prod.data.view()) == g["prod"]
    assert digest(ckks.ckks_multiply(ctx, cx, cy, mode="unfused").data.view()) == g["prod"]
    assert digest(ckks.ckks_square(ctx, cx).data.view()) == g["square"]
    kb, ka = key_switch(ctx, cy.data.view()[1], c1["rlk"])
    assert digest(kb) == g["ks_b"] and digest(ka) == g["ks_a"]
    lin = ckks.ckks_relinearize(ctx, prod, c1["rlk"])
    assert digest(lin.data.view()) == g["relin"]
    res = ckks.ckks_rescale(ctx, lin)
    assert digest(res.data.view()) == g["rescale"]
    assert res.scale == g["rescale_scale"]
    gks = c1["gks"]
    assert digest(ckks.ckks_rotate(ctx, cx, 1, gks).data.view()) == g["rot1"]
    assert digest(ckks.ckks_rotate(ctx, cx, 5, gks).data.view()) == g["rot5"]
    assert digest(ckks.ckks_conjugate(ctx, cx, gks).data.view()) == g["conj"]
    q_last = ctx.q_values[-1]
    boosted = ckks.ckks_rescale(ctx, ckks.ckks_rotate(
        ctx, ckks.ckks_multiply_scalar(ctx, cx, 1.0, scale=float(q_last)), 1, gks))
    assert digest(boosted.data.view()) == g["boosted_rot"]
    # decode runs the same float64 host path on identical residues
    arr = golden_arrays["ckks_c1"]
    dec = ckks.ckks_decode(ctx, ckks.ckks_decrypt(ctx, res, sk))
    assert np.array_equal(dec, arr["dec_mul"])
    assert np.max(np.abs(dec - x * y)) == pytest.approx(g["err_mul"])
    dec_rot = ckks.ckks_decode(ctx, ckks.ckks_decrypt(ctx, boosted, sk))
    assert np.array_equal(dec_rot, arr["dec_rot"])


def test_small_key_switch_full_arrays(golden_arrays):
    from paper_2503_22227_b200.context import Context, EncryptionParams, Scheme
    from paper_2503_22227_b200.coremath.primes import gen_ntt_prime_chain
    from paper_2503_22227_b200.keys import key_switch, keygen, relin_keygen

    s = golden_arrays["small"]
    moduli = tuple(m.value for m in gen_ntt_prime_chain(36, 64, 3))
    ctx = Context(EncryptionParams(Scheme.CKKS, 64, moduli, default_scale=float(1 << 35)))
    sk = keygen(ctx, seeded_rng(5))
    assert (to_u64(sk.s.view()) == s["ks_sk"]).all()
    rk = relin_keygen(ctx, sk, seeded_rng(9))
    assert (np.stack([to_u64(d.view()) for d in rk.digits]) == s["ks_rlk"]).all()
    d = ctx.ntt_chain.forward(seeded_rng(11).uniform_residues(ctx.q_arr(), ctx.n),
                              np.arange(3))
    assert (d == s["ks_d"]).all()
    b, a = key_switch(ctx, d, rk)
    assert (to_u64(b) == s["ks_b"]).all()
    assert (to_u64(a) == s["ks_a"]).all()
