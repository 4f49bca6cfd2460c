"""CATF wire-record goldens: records written by the REFERENCE's own
serializer (rnsfhe/serial.py) for n = 64 objects built from fixed seeds.
Run in the build container (needs /root/reference):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_serial_golden.py

Output: tests/golden/serial.json (record bytes as hex).  tests/test_gpu_serial.py
rebuilds the same objects on the B200 and checks its records byte for byte.
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

from rnsfhe import serial  # noqa: E402
from rnsfhe.context import Context, EncryptionParams, Scheme  # noqa: E402
from rnsfhe.coremath.primes import gen_ntt_prime_chain  # noqa: E402
from rnsfhe.coremath.sampling import Rng  # noqa: E402
from rnsfhe.keys import galois_keygen, keygen, pk_gen, relin_keygen  # noqa: E402
from rnsfhe.schemes import bgv, ckks  # noqa: E402


def seeded(s):
    return Rng(int(s).to_bytes(32, "little"))


def main():
    out = {}
    n = 64
    moduli = tuple(m.value for m in gen_ntt_prime_chain(36, n, 3))
    for scheme in (Scheme.CKKS, Scheme.BGV):
        if scheme is Scheme.CKKS:
            params = EncryptionParams(scheme, n, moduli, default_scale=float(1 << 35))
        else:
            params = EncryptionParams(scheme, n, moduli, plain_modulus=65537)
        ctx = Context(params)
        sk = keygen(ctx, seeded(1))
        pk = pk_gen(ctx, sk, seeded(2))
        rlk = relin_keygen(ctx, sk, seeded(3))
        gks = galois_keygen(ctx, sk, [1], seeded(4), include_conj=True)
        tag = scheme.value
        rec = {"params": serial.serialize_params(params).hex(),
               "sk": serial.serialize_secret_key(params, sk).hex(),
               "pk": serial.serialize_public_key(params, pk).hex(),
               "pk_seeded": serial.serialize_public_key(params, pk, seeded=True).hex(),
               "relin": serial.serialize_kswitch_key(params, rlk).hex(),
               "galois": serial.serialize_galois_keys(params, gks).hex()}
        if scheme is Scheme.CKKS:
            x = np.random.default_rng(1).uniform(-1, 1, n // 2)
            ct = ckks.ckks_encrypt(ctx, ckks.ckks_encode(ctx, x), pk, seeded(10))
            rec["ct"] = serial.serialize_block(params, serial.KIND_CIPHERTEXT, ct.data,
                                               scale=ct.scale).hex()
        else:
            va = np.random.default_rng(7).integers(0, 65537, 64, dtype=np.uint64)
            ct = bgv.bgv_encrypt_ints(ctx, va, pk, seeded(10))
            rec["ct"] = serial.serialize_block(params, serial.KIND_CIPHERTEXT, ct.data,
                                               aux=ct.plain_factor).hex()
        out[tag] = rec
    with open(os.path.join(HERE, "serial.json"), "w") as f:
        json.dump(out, f, indent=0)


if __name__ == "__main__":
    main()
