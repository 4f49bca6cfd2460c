"""Host parts of the CATF wire format (paper_2503_22227_b200/serial.py):
parameter records byte-identical to the reference's own serializer
(tests/golden/serial.json, written by the reference), crc32_combine equal
to zlib, and the parser's error behaviour (reference serial.py:80-127)."""
import json
import os
import zlib

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def gold():
    with open(os.path.join(HERE, "golden", "serial.json")) as f:
        return json.load(f)


def _params(scheme):
    from paper_2503_22227_b200.context import EncryptionParams, Scheme
    from paper_2503_22227_b200.coremath.primes import gen_ntt_prime_chain

    moduli = tuple(m.value for m in gen_ntt_prime_chain(36, 64, 3))
    if scheme == "ckks":
        return EncryptionParams(Scheme.CKKS, 64, moduli, default_scale=float(1 << 35))
    return EncryptionParams(Scheme.BGV, 64, moduli, plain_modulus=65537)


@pytest.mark.parametrize("scheme", ["ckks", "bgv"])
def test_params_record_matches_reference(scheme, gold):
    from paper_2503_22227_b200 import serial

    p = _params(scheme)
    assert serial.serialize_params(p).hex() == gold[scheme]["params"]
    back = serial.deserialize_params(bytes.fromhex(gold[scheme]["params"]))
    assert (back.scheme, back.n, tuple(back.coeff_moduli)) == (p.scheme, p.n, tuple(p.coeff_moduli))
    assert back.plain_modulus == p.plain_modulus and back.default_scale == p.default_scale


def test_crc32_combine_equals_zlib():
    from paper_2503_22227_b200.serial import crc32_combine

    rng = np.random.default_rng(0)
    for la, lb in ((0, 0), (1, 0), (0, 5), (13, 4096), (4097, 3), (100000, 77777)):
        a = rng.integers(0, 256, la, dtype=np.uint8).tobytes()
        b = rng.integers(0, 256, lb, dtype=np.uint8).tobytes()
        assert crc32_combine(zlib.crc32(a), zlib.crc32(b), lb) == zlib.crc32(a + b)


def test_parser_rejects_corruption(gold):
    from paper_2503_22227_b200 import serial

    rec = bytearray(bytes.fromhex(gold["ckks"]["sk"]))
    parsed = serial.parse_record(bytes(rec), serial.KIND_SK)
    assert parsed.n == 64 and parsed.level == 3 and len(parsed.body) == 8 * 64
    bad = bytearray(rec)
    bad[100] ^= 1
    with pytest.raises(serial.SerializationError, match="checksum"):
        serial.parse_record(bytes(bad))
    with pytest.raises(serial.SerializationError, match="truncated"):
        serial.parse_record(bytes(rec[:-10]))
    bad = bytearray(rec)
    bad[0:4] = b"XXXX"
    with pytest.raises(serial.SerializationError, match="magic"):
        serial.parse_record(bytes(bad))
    with pytest.raises(serial.SerializationError, match="expected kind"):
        serial.parse_record(bytes(rec), serial.KIND_PK)
