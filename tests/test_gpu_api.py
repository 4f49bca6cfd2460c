"""Operator-surface behaviour on the device, mirroring the reference
test-suite (tests/test_ckks.py, test_bgv.py, test_bfv.py): error semantics,
fused == unfused, square == multiply, slot-permutation rotations, depth-two
chains, exact BFV/BGV arithmetic mod t, pool statistics on the HBM arena."""

import numpy as np
import pytest

from fhe_testutil import seeded_rng, to_u64

pytestmark = pytest.mark.gpu

N = 64
HALF = N // 2


@pytest.fixture(scope="module")
def ck():
    from paper_2503_22227_b200.context import Context, EncryptionParams, Scheme
    from paper_2503_22227_b200.coremath.primes import gen_ntt_prime_chain
    from paper_2503_22227_b200.keys import galois_keygen, keygen, pk_gen, relin_keygen

    qs = tuple(m.value for m in gen_ntt_prime_chain(36, N, 3))
    ctx = Context(EncryptionParams(Scheme.CKKS, N, qs, default_scale=float(1 << 35)))
    sk = keygen(ctx, seeded_rng(1))
    return {"ctx": ctx, "sk": sk, "pk": pk_gen(ctx, sk, seeded_rng(2)),
            "rlk": relin_keygen(ctx, sk, seeded_rng(3)),
            "gks": galois_keygen(ctx, sk, [1, 3, -1], seeded_rng(4), include_conj=True)}


def slots(rng):
    return rng.uniform(-1, 1, HALF) + 1j * rng.uniform(-1, 1, HALF)


def test_ckks_error_semantics(ck):
    from paper_2503_22227_b200.coremath.modmath import ParameterError
    from paper_2503_22227_b200.schemes import ckks

    ctx, pk = ck["ctx"], ck["pk"]
    a = slots(np.random.default_rng(1))
    ca = ckks.ckks_encrypt(ctx, ckks.ckks_encode(ctx, a), pk, seeded_rng(22))
    low = ckks.ckks_rescale(ctx, ckks.ckks_multiply_plain(ctx, ca, ckks.ckks_encode(ctx, a)))
    with pytest.raises(ckks.LevelMismatch):
        ckks.ckks_add(ctx, ca, low)
    off = ckks.ckks_encrypt(ctx, ckks.ckks_encode(ctx, a, scale=2.0 ** 20), pk, seeded_rng(23))
    with pytest.raises(ckks.ScaleMismatch):
        ckks.ckks_add(ctx, ca, off)
    lvl1 = ckks.ckks_rescale(ctx, low)
    with pytest.raises(ckks.LevelMismatch):
        ckks.ckks_rescale(ctx, lvl1)
    with pytest.raises(ckks.EncodeRangeError):
        ckks.ckks_encode(ctx, np.full(HALF, 1e30))
    with pytest.raises(ParameterError):
        ckks.ckks_encode(ctx, np.zeros(HALF + 1))
    with pytest.raises(ParameterError):
        ckks.ckks_multiply(ctx, ca, ca, mode="bogus")


def test_ckks_algebra(ck):
    from paper_2503_22227_b200.schemes import ckks

    ctx, pk, sk = ck["ctx"], ck["pk"], ck["sk"]
    rng = np.random.default_rng(2)
    a, b, c = slots(rng), slots(rng), slots(rng)
    ca = ckks.ckks_encrypt(ctx, ckks.ckks_encode(ctx, a), pk, seeded_rng(13))
    cb = ckks.ckks_encrypt(ctx, ckks.ckks_encode(ctx, b), pk, seeded_rng(14))
    dec = lambda ct: ckks.ckks_decode(ctx, ckks.ckks_decrypt(ctx, ct, sk))  # noqa: E731
    assert np.max(np.abs(dec(ckks.ckks_add(ctx, ca, cb)) - (a + b))) < 2e-4
    assert np.max(np.abs(dec(ckks.ckks_sub(ctx, ca, cb)) - (a - b))) < 2e-4
    assert np.max(np.abs(dec(ckks.ckks_add_plain(ctx, ca, ckks.ckks_encode(ctx, b))) - (a + b))) < 2e-4
    fused = ckks.ckks_multiply(ctx, ca, cb)
    assert (to_u64(fused.data.view()) ==
            to_u64(ckks.ckks_multiply(ctx, ca, cb, mode="unfused").data.view())).all()
    assert (to_u64(ckks.ckks_square(ctx, ca).data.view()) ==
            to_u64(ckks.ckks_multiply(ctx, ca, ca).data.view())).all()
    ab = ckks.ckks_rescale(ctx, ckks.ckks_relinearize(ctx, fused, ck["rlk"]))
    pc = ckks.ckks_encode(ctx, c, scale=ab.scale, level=ab.level)
    abc = ckks.ckks_rescale(ctx, ckks.ckks_multiply_plain(ctx, ab, pc))
    assert abc.level == 1
    assert np.max(np.abs(dec(abc) - a * b * c)) < 1e-2
    z = 0.5 - 0.25j
    scaled = ckks.ckks_rescale(ctx, ckks.ckks_multiply_scalar(ctx, ca, z))
    assert np.max(np.abs(dec(scaled) - a * z)) < 1e-3


def test_rotation_is_slot_permutation(ck):
    from paper_2503_22227_b200.keys import automorph_rows
    from paper_2503_22227_b200.schemes import ckks

    ctx = ck["ctx"]
    a = slots(np.random.default_rng(3))
    pt = ckks.ckks_encode(ctx, a)
    perm = automorph_rows(ctx, pt.data.view()[0].contiguous(), ctx.galois_elt_for_step(1))
    pt.data.view()[0].copy_(perm)
    assert np.max(np.abs(ckks.ckks_decode(ctx, pt) - np.roll(a, -1))) < 1e-6
    host = ctx.galois_perm(ctx.galois_elt_for_step(1))
    orig = to_u64(ckks.ckks_encode(ctx, a).data.view()[0])
    assert (to_u64(perm) == orig[:, host]).all()


def test_pool_statistics_on_device(ck):
    from paper_2503_22227_b200.schemes import ckks

    ctx = ck["ctx"]
    before = ctx.pool.pool_stats()["ask_count"]
    a = slots(np.random.default_rng(4))
    ca = ckks.ckks_encrypt(ctx, ckks.ckks_encode(ctx, a), ck["pk"], seeded_rng(30))
    for _ in range(4):
        ckks.ckks_relinearize(ctx, ckks.ckks_multiply(ctx, ca, ca), ck["rlk"])
    st = ctx.pool.pool_stats()
    assert st["ask_count"] > before and st["reuse_count"] > 0
    assert st["high_water_bytes"] <= st["capacity"] + st["overflow_count"] * (1 << 30)


@pytest.mark.parametrize("scheme", ["bgv", "bfv"])
def test_exact_integer_ops(scheme):
    from paper_2503_22227_b200.context import Context, EncryptionParams, Scheme
    from paper_2503_22227_b200.coremath.primes import gen_ntt_prime_chain
    from paper_2503_22227_b200.keys import galois_keygen, keygen, pk_gen, relin_keygen
    from paper_2503_22227_b200.schemes import bfv, bgv
    from paper_2503_22227_b200.schemes.batching import batch_decode, batch_encode

    T = 65537
    mod = bgv if scheme == "bgv" else bfv
    qs = tuple(m.value for m in gen_ntt_prime_chain(36, N, 3))
    ctx = Context(EncryptionParams(Scheme(scheme), N, qs, plain_modulus=T))
    sk = keygen(ctx, seeded_rng(1))
    pk = pk_gen(ctx, sk, seeded_rng(2))
    rlk = relin_keygen(ctx, sk, seeded_rng(3))
    gks = galois_keygen(ctx, sk, [1], seeded_rng(4), include_conj=True)
    rng = np.random.default_rng(9)
    a = rng.integers(0, T, N, dtype=np.uint64)
    b = rng.integers(0, T, N, dtype=np.uint64)
    enc = getattr(mod, f"{scheme}_encrypt_ints")
    dec = lambda ct: batch_decode(ctx, getattr(mod, f"{scheme}_decrypt")(ctx, ct, sk))  # noqa
    ca, cb = enc(ctx, a, pk, seeded_rng(10)), enc(ctx, b, pk, seeded_rng(11))
    ao, bo = a.astype(object), b.astype(object)
    assert dec(getattr(mod, f"{scheme}_add")(ctx, ca, cb)).tolist() == ((ao + bo) % T).tolist()
    assert dec(getattr(mod, f"{scheme}_sub")(ctx, ca, cb)).tolist() == ((ao - bo) % T).tolist()
    sq = getattr(mod, f"{scheme}_relinearize")(ctx, getattr(mod, f"{scheme}_square")(ctx, ca), rlk)
    assert dec(sq).tolist() == (ao * ao % T).tolist()
    mp = getattr(mod, f"{scheme}_multiply_plain")(ctx, ca, batch_encode(ctx, b))
    assert dec(mp).tolist() == (ao * bo % T).tolist()
    swapped = getattr(mod, f"{scheme}_rotate_columns")(ctx, ca, gks)
    assert dec(swapped).tolist() == np.concatenate([a[HALF:], a[:HALF]]).tolist()
    rot = getattr(mod, f"{scheme}_rotate_rows")(ctx, ca, 1, gks)
    want = np.concatenate([np.roll(a[:HALF], -1), np.roll(a[HALF:], -1)])
    assert dec(rot).tolist() == want.tolist()
    if scheme == "bgv":
        ms = bgv.bgv_mod_switch(ctx, sq)
        assert dec(ms).tolist() == (ao * ao % T).tolist()
        mixed = bgv.bgv_add(ctx, ms, bgv.bgv_mod_switch(ctx, cb))
        assert dec(mixed).tolist() == ((ao * ao + bo) % T).tolist()
        assert bgv.bgv_noise_budget(ctx, ca, sk) > 10
    else:
        assert bfv.noise_budget(ctx, ca, sk) > 10


def test_host_batch_pipeline_matches_operators(ck):
    """host_io.hmult_relin_host_batch (H2D / compute / D2H on three streams)
    returns the same residues as the operators run one by one."""
    import torch

    from paper_2503_22227_b200.host_io import CopyStreams, hmult_relin_host_batch
    from paper_2503_22227_b200.schemes import ckks

    ctx, pk, rlk = ck["ctx"], ck["pk"], ck["rlk"]
    rng = np.random.default_rng(11)
    cts = [ckks.ckks_encrypt(ctx, ckks.ckks_encode(ctx, slots(rng)), pk, seeded_rng(20 + i))
           for i in range(6)]
    level = cts[0].level
    hx = torch.stack([c.data.view().cpu() for c in cts[0::2]]).pin_memory()
    hy = torch.stack([c.data.view().cpu() for c in cts[1::2]]).pin_memory()
    out = torch.empty_like(hx).pin_memory()
    streams = CopyStreams.create()
    for _ in range(2):  # second round reuses pool blocks across streams
        hmult_relin_host_batch(ctx, hx, hy, cts[0].scale, cts[1].scale, level, rlk, out, streams)
    torch.cuda.synchronize()
    for b in range(3):
        want = ckks.ckks_relinearize(ctx, ckks.ckks_multiply(ctx, cts[2 * b], cts[2 * b + 1]), rlk)
        assert torch.equal(out[b], want.data.view().cpu())
