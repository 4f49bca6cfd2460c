"""CATF wire records of device-resident objects (serial.py): byte-identical
to the reference's serializer on the same seeded objects (tests/golden/
serial.json), round trips, the zero-copy pinned path at config-4 size, and
the device CRC-32 (fhe_crc32) equal to zlib on awkward lengths."""
import json
import os
import zlib

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def gold():
    with open(os.path.join(HERE, "golden", "serial.json")) as f:
        return json.load(f)


def _objects(scheme):
    from paper_2503_22227_b200.context import Context, EncryptionParams, PoolConfig, Scheme
    from paper_2503_22227_b200.coremath.primes import gen_ntt_prime_chain
    from paper_2503_22227_b200.coremath.sampling import Rng
    from paper_2503_22227_b200.keys import galois_keygen, keygen, pk_gen, relin_keygen
    from paper_2503_22227_b200.schemes import bgv, ckks

    seeded = lambda s: Rng(int(s).to_bytes(32, "little"))  # noqa: E731
    n = 64
    moduli = tuple(m.value for m in gen_ntt_prime_chain(36, n, 3))
    if scheme == "ckks":
        params = EncryptionParams(Scheme.CKKS, n, moduli, default_scale=float(1 << 35))
    else:
        params = EncryptionParams(Scheme.BGV, n, moduli, plain_modulus=65537)
    ctx = Context(params, PoolConfig(unit_mb=8, cap_mb=64))
    sk = keygen(ctx, seeded(1))
    pk = pk_gen(ctx, sk, seeded(2))
    rlk = relin_keygen(ctx, sk, seeded(3))
    gks = galois_keygen(ctx, sk, [1], seeded(4), include_conj=True)
    if scheme == "ckks":
        x = np.random.default_rng(1).uniform(-1, 1, n // 2)
        ct = ckks.ckks_encrypt(ctx, ckks.ckks_encode(ctx, x), pk, seeded(10))
    else:
        va = np.random.default_rng(7).integers(0, 65537, 64, dtype=np.uint64)
        ct = bgv.bgv_encrypt_ints(ctx, va, pk, seeded(10))
    return ctx, params, sk, pk, rlk, gks, ct


@pytest.mark.parametrize("scheme", ["ckks", "bgv"])
def test_records_byte_identical_to_reference(scheme, gold):
    import torch

    from paper_2503_22227_b200 import serial

    ctx, params, sk, pk, rlk, gks, ct = _objects(scheme)
    g = gold[scheme]
    assert serial.serialize_secret_key(params, sk).hex() == g["sk"]
    assert serial.serialize_public_key(params, pk).hex() == g["pk"]
    assert serial.serialize_public_key(params, pk, seeded=True).hex() == g["pk_seeded"]
    assert serial.serialize_kswitch_key(params, rlk).hex() == g["relin"]
    assert serial.serialize_galois_keys(params, gks).hex() == g["galois"]
    aux = int(getattr(ct, "plain_factor", 0) or 0)
    got = serial.serialize_block(params, serial.KIND_CIPHERTEXT, ct.data,
                                 scale=float(getattr(ct, "scale", 0.0) or 0.0), aux=aux)
    assert got.hex() == g["ct"]
    # round trips from the reference's bytes
    cd, rec = serial.deserialize_block(params, bytes.fromhex(g["ct"]), serial.KIND_CIPHERTEXT, ctx)
    assert torch.equal(cd.view(), ct.data.view()) and rec.aux == aux
    pk2 = serial.deserialize_public_key(ctx, bytes.fromhex(g["pk_seeded"]))
    assert torch.equal(pk2.data.view(), pk.data.view())
    sk2 = serial.deserialize_secret_key(ctx, bytes.fromhex(g["sk"]))
    assert torch.equal(sk2.s.view(), sk.s.view())
    r2 = serial.deserialize_kswitch_key(ctx, bytes.fromhex(g["relin"]))
    assert torch.equal(r2.data.view(), rlk.data.view())
    g2 = serial.deserialize_galois_keys(ctx, bytes.fromhex(g["galois"]))
    assert sorted(g2.keys) == sorted(gks.keys)
    for e in gks.keys:
        assert torch.equal(g2.keys[e].data.view(), gks.keys[e].data.view())
    bad = bytearray(bytes.fromhex(g["ct"]))
    bad[len(bad) // 2] ^= 0x40
    with pytest.raises(serial.SerializationError, match="checksum"):
        serial.deserialize_block(params, bytes(bad), serial.KIND_CIPHERTEXT, ctx)


def test_device_crc32_matches_zlib():
    import torch

    from paper_2503_22227_b200.serial import device_crc32

    rng = np.random.default_rng(5)
    for nb in (0, 1, 7, 4095, 4096, 4097, 3 * 4096 + 5, 10_000_003):
        a = rng.integers(0, 256, nb, dtype=np.uint8)
        t = torch.from_numpy(a).cuda()
        assert device_crc32(t) == zlib.crc32(a.tobytes()), nb


def test_zero_copy_config4_ciphertext_round_trip():
    import torch

    from paper_2503_22227_b200 import serial
    from paper_2503_22227_b200.context import Context, PoolConfig, hybrid_params
    from paper_2503_22227_b200.rnspoly import CData, Domain

    ctx = Context(hybrid_params(1 << 16, 30, special=10, dnum=3, scale=float(2 ** 49)),
                  PoolConfig(unit_mb=64, cap_mb=1024))
    words = torch.randint(0, 1 << 49, (2, 30, 1 << 16), dtype=torch.int64, device="cuda")
    cd = CData.wrap(words.reshape(-1), 2, 30, 1 << 16, Domain.EVALUATION)
    buf = torch.empty(40 << 20, dtype=torch.uint8).pin_memory()
    mv = serial.serialize_block_into(ctx.params, serial.KIND_CIPHERTEXT, cd, scale=2.0 ** 49,
                                     buf=buf)
    raw = bytes(mv)
    rec = serial.parse_record(raw, serial.KIND_CIPHERTEXT)  # host zlib verification
    assert rec.level == 30 and rec.size_poly == 2 and rec.scale == 2.0 ** 49
    cd2, _ = serial.deserialize_block(ctx.params, mv, serial.KIND_CIPHERTEXT, ctx)
    assert torch.equal(cd2.view(), words)
