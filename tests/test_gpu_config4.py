"""Config 4 at full size (N=2^16, L=30) on the B200.

* reference gadget (alpha=1, K=0): keys, ciphertexts, product, relinearised
  and rescaled ciphertexts bit-identical to the reference's own run
  (tests/golden/digests.json "ckks_c4", MAX_CHAIN_LEN patched to 30 exactly
  as the reference needs);
* hybrid dnum=3 (alpha=10, K=10 x 60-bit): bit-exact against the C oracle's
  restatement (oracle/c/fhe_oracle.c) and decryption error within the
  tolerance of BASELINE.md: max|dec - x*y| <= reference error + 2^-20.
"""

import numpy as np
import pytest

from fhe_testutil import digest, seeded_rng

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


@pytest.fixture(scope="module")
def ref_gadget(golden):
    import paper_2503_22227_b200.context as pctx
    from paper_2503_22227_b200.context import Context, EncryptionParams, PoolConfig, Scheme

    g = golden["ckks_c4"]
    old = pctx.MAX_CHAIN_LEN
    pctx.MAX_CHAIN_LEN = 30
    try:
        primes = tuple(int(p) for p in g["primes"])
        ctx = Context(EncryptionParams(Scheme.CKKS, 1 << 16, primes, default_scale=g["scale"]),
                      PoolConfig(unit_mb=200, cap_mb=4096))
    finally:
        pctx.MAX_CHAIN_LEN = old
    return g, ctx


def test_reference_gadget_bit_identical_at_config4(ref_gadget):
    from paper_2503_22227_b200.keys import keygen, pk_gen, relin_keygen
    from paper_2503_22227_b200.schemes import ckks

    g, ctx = ref_gadget
    sk = keygen(ctx, seeded_rng(4))
    assert digest(sk.s.view()) == g["sk_s"]
    pk = pk_gen(ctx, sk, seeded_rng(41))
    rlk = relin_keygen(ctx, sk, seeded_rng(42))
    assert digest(rlk.digits[0].view()) == g["rlk0"]
    assert digest(rlk.digits[29].view()) == g["rlk29"]
    vr = np.random.default_rng(9)
    x = vr.uniform(-1, 1, ctx.n // 2)
    y = vr.uniform(-1, 1, ctx.n // 2)
    cx = ckks.ckks_encrypt(ctx, ckks.ckks_encode(ctx, x), pk, seeded_rng(43))
    cy = ckks.ckks_encrypt(ctx, ckks.ckks_encode(ctx, y), pk, seeded_rng(44))
    assert digest(cx.data.view()) == g["ct_x"] and digest(cy.data.view()) == g["ct_y"]
    prod = ckks.ckks_multiply(ctx, cx, cy)
    assert digest(prod.data.view()) == g["prod"]
    lin = ckks.ckks_relinearize(ctx, prod, rlk)
    assert digest(lin.data.view()) == g["relin"]
    res = ckks.ckks_rescale(ctx, lin)
    assert digest(res.data.view()) == g["rescale"]


@pytest.fixture(scope="module", params=[50, 60], ids=["P50_fp64", "P60_int"])
def hybrid(request):
    """P = 10 x 50-bit (FP64-pipe NTT path) and 10 x 60-bit (integer path)."""
    from paper_2503_22227_b200.context import Context, PoolConfig, hybrid_params
    from paper_2503_22227_b200.keys import galois_keygen, keygen, pk_gen, relin_keygen

    params = hybrid_params(1 << 16, 30, bits=50, special=10, special_bits=request.param,
                           dnum=3, scale=float(2 ** 49))
    ctx = Context(params, PoolConfig(unit_mb=200, cap_mb=4096))
    sk = keygen(ctx, seeded_rng(4))
    return {"ctx": ctx, "sk": sk, "pk": pk_gen(ctx, sk, seeded_rng(41)),
            "rlk": relin_keygen(ctx, sk, seeded_rng(42)),
            "gks": galois_keygen(ctx, sk, [1], seeded_rng(45))}


def test_hybrid_hmult_relin_rescale_bit_exact_vs_oracle(hybrid, golden):
    from oracle import fast
    from paper_2503_22227_b200.schemes import ckks

    ctx, sk = hybrid["ctx"], hybrid["sk"]
    vr = np.random.default_rng(9)
    x = vr.uniform(-1, 1, ctx.n // 2)
    y = vr.uniform(-1, 1, ctx.n // 2)
    cx = ckks.ckks_encrypt(ctx, ckks.ckks_encode(ctx, x), hybrid["pk"], seeded_rng(43))
    cy = ckks.ckks_encrypt(ctx, ckks.ckks_encode(ctx, y), hybrid["pk"], seeded_rng(44))
    lin = ckks.ckks_relinearize(ctx, ckks.ckks_multiply(ctx, cx, cy), hybrid["rlk"])
    res = ckks.ckks_rescale(ctx, lin)
    Q, P = ctx.q_values, ctx.special_values
    d0, d1, d2 = fast.tensor(cx.data.to_numpy(), cy.data.to_numpy(), Q)
    keys = hybrid["rlk"].data.to_numpy().reshape(3, 2, 40, ctx.n)
    kb, ka = fast.key_switch(d2, keys, Q, alpha=ctx.ks_alpha, special=P)
    want = np.stack([fast.add(d0, kb, Q), fast.add(d1, ka, Q)])
    assert np.array_equal(lin.data.to_numpy(), want)
    assert np.array_equal(res.data.to_numpy(), fast.rescale(want, Q))
    dec = ckks.ckks_decode(ctx, ckks.ckks_decrypt(ctx, res, sk))
    err = float(np.max(np.abs(dec - x * y)))
    # tolerance: reference error at these parameters + 2^-20
    assert err <= golden["ckks_c4"]["err_mul"] + 2.0 ** -20, err


def test_fused_hmult_relin_bit_exact(hybrid):
    """fhe_hmult_relin (tensor product formed inside the key switch's finishing
    kernel) gives the words of ckks_multiply + ckks_relinearize: full level,
    squaring, and a batch of 3 at a lower level (ragged last digit)."""
    import torch

    from paper_2503_22227_b200.keys import hmult_relin_into
    from paper_2503_22227_b200.schemes import ckks

    ctx, rlk = hybrid["ctx"], hybrid["rlk"]
    vr = np.random.default_rng(19)
    cts = [ckks.ckks_encrypt(ctx, ckks.ckks_encode(ctx, vr.uniform(-1, 1, ctx.n // 2)),
                             hybrid["pk"], seeded_rng(60 + i)) for i in range(4)]
    want = ckks.ckks_relinearize(ctx, ckks.ckks_multiply(ctx, cts[0], cts[1]), rlk)
    got = ckks.ckks_multiply_relinearize(ctx, cts[0], cts[1], rlk)
    assert got.scale == want.scale and got.level == want.level
    assert torch.equal(got.data.view(), want.data.view())
    sq_want = ckks.ckks_relinearize(ctx, ckks.ckks_square(ctx, cts[2]), rlk)
    sq_got = ckks.ckks_multiply_relinearize(ctx, cts[2], None, rlk)
    assert torch.equal(sq_got.data.view(), sq_want.data.view())
    # batch of 3 pairs at level 17 (digits 10 + 7), stacked (B, 2, level, n)
    lv = 17
    low = [ckks.CkksCiphertext(ckks.CData.wrap(c.data.view()[:, :lv].contiguous().reshape(-1), 2,
                                               lv, ctx.n, ckks.Domain.EVALUATION), c.scale, lv)
           for c in cts]
    X = torch.stack([low[i].data.view() for i in (0, 1, 2)])
    Y = torch.stack([low[i].data.view() for i in (3, 0, 1)])
    out = torch.empty_like(X)
    hmult_relin_into(ctx, lv, X, Y, rlk, out[:, 0], out[:, 1], batch=3)
    for b, (i, j) in enumerate(((0, 3), (1, 0), (2, 1))):
        ref = ckks.ckks_relinearize(ctx, ckks.ckks_multiply(ctx, low[i], low[j]), rlk)
        assert torch.equal(out[b], ref.data.view()), b


def test_hybrid_boosted_rotate_within_tolerance(hybrid):
    from paper_2503_22227_b200.schemes import ckks

    ctx, sk = hybrid["ctx"], hybrid["sk"]
    vr = np.random.default_rng(11)
    x = vr.uniform(-1, 1, ctx.n // 2)
    cx = ckks.ckks_encrypt(ctx, ckks.ckks_encode(ctx, x), hybrid["pk"], seeded_rng(46))
    boosted = ckks.ckks_multiply_scalar(ctx, cx, 1.0, scale=float(ctx.q_values[-1]))
    rot = ckks.ckks_rescale(ctx, ckks.ckks_rotate(ctx, boosted, 1, hybrid["gks"]))
    dec = ckks.ckks_decode(ctx, ckks.ckks_decrypt(ctx, rot, sk))
    # reference boosted-rotate error at config 4 is 2^-23.2
    assert float(np.max(np.abs(dec - np.roll(x, -1)))) <= 2.0 ** -23.2 + 2.0 ** -20
    # plain rotation is exact-permutation of slots up to key-switch noise: with
    # hybrid key switching the noise is small enough even without boosting
    plain = ckks.ckks_rotate(ctx, cx, 1, hybrid["gks"])
    dec2 = ckks.ckks_decode(ctx, ckks.ckks_decrypt(ctx, plain, sk))
    assert float(np.max(np.abs(dec2 - np.roll(x, -1)))) < 1e-6


def test_fused_moddown_finish_matches_separate_pass():
    """The opt-in ModDown finish fused into the conversion NTT's epilogue
    (FHE_FUSE_MODDOWN=1) gives the same relinearized words as the separate
    finish pass (child processes: the switch is read once per process)."""
    import hashlib
    import os
    import subprocess
    import sys

    code = r'''
import hashlib, numpy as np, torch
from paper_2503_22227_b200.context import Context, PoolConfig, hybrid_params
from paper_2503_22227_b200.coremath.sampling import Rng
from paper_2503_22227_b200.keys import keygen, pk_gen, relin_keygen
from paper_2503_22227_b200.schemes import ckks
ctx = Context(hybrid_params(1 << 16, 30, bits=50, special=10, special_bits=50, dnum=3,
                            scale=float(2 ** 49)), PoolConfig(unit_mb=200, cap_mb=4096))
seed = lambda s: Rng(int(s).to_bytes(32, "little"))
sk = keygen(ctx, seed(4)); pk = pk_gen(ctx, sk, seed(41)); rlk = relin_keygen(ctx, sk, seed(42))
r = np.random.default_rng(9)
x = ckks.ckks_encrypt(ctx, ckks.ckks_encode(ctx, r.uniform(-1, 1, ctx.n // 2)), pk, seed(43))
y = ckks.ckks_encrypt(ctx, ckks.ckks_encode(ctx, r.uniform(-1, 1, ctx.n // 2)), pk, seed(44))
out = ckks.ckks_relinearize(ctx, ckks.ckks_multiply(ctx, x, y), rlk)
print(hashlib.sha256(out.data.view().cpu().numpy().tobytes()).hexdigest())
'''
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    digests = []
    for flag in ("0", "1"):
        env = dict(os.environ, FHE_FUSE_MODDOWN=flag, PYTHONPATH=root)
        out = subprocess.run([sys.executable, "-c", code], env=env, cwd=root, capture_output=True,
                             text=True, timeout=900)
        assert out.returncode == 0, out.stderr[-2000:]
        digests.append(out.stdout.strip().splitlines()[-1])
    assert digests[0] == digests[1]
    del hashlib


def test_fused_hmult_relin_switches():
    """fhe_hmult_relin with the tensor formed inside the finishing kernel
    (FHE_HMULT_TENS=1), with the default materialised tensor, and with the
    fused inner/finish kernel disabled (FHE_FUSE_INNER_FINISH=0, the TENS
    request then falls back): every product and square is the same words as
    ckks_multiply/ckks_square + ckks_relinearize."""
    import os
    import subprocess
    import sys

    code = r'''
import hashlib, numpy as np, torch
from paper_2503_22227_b200.context import Context, PoolConfig, hybrid_params
from paper_2503_22227_b200.coremath.sampling import Rng
from paper_2503_22227_b200.keys import keygen, pk_gen, relin_keygen
from paper_2503_22227_b200.schemes import ckks
ctx = Context(hybrid_params(1 << 16, 30, bits=50, special=10, special_bits=50, dnum=3,
                            scale=float(2 ** 49)), PoolConfig(unit_mb=200, cap_mb=4096))
seed = lambda s: Rng(int(s).to_bytes(32, "little"))
sk = keygen(ctx, seed(4)); pk = pk_gen(ctx, sk, seed(41)); rlk = relin_keygen(ctx, sk, seed(42))
r = np.random.default_rng(9)
x = ckks.ckks_encrypt(ctx, ckks.ckks_encode(ctx, r.uniform(-1, 1, ctx.n // 2)), pk, seed(43))
y = ckks.ckks_encrypt(ctx, ckks.ckks_encode(ctx, r.uniform(-1, 1, ctx.n // 2)), pk, seed(44))
a = ckks.ckks_relinearize(ctx, ckks.ckks_multiply(ctx, x, y), rlk)
b = ckks.ckks_multiply_relinearize(ctx, x, y, rlk)
c = ckks.ckks_relinearize(ctx, ckks.ckks_square(ctx, x), rlk)
d = ckks.ckks_multiply_relinearize(ctx, x, None, rlk)
h = lambda c: hashlib.sha256(c.data.view().cpu().numpy().tobytes()).hexdigest()
assert h(a) == h(b) and h(c) == h(d)
print(h(a), h(c))
'''
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    digests = set()
    # (fused finish, tensor terms in the finish, cp.async-staged finish kernel)
    for fin, tens, staged in (("1", "1", "1"), ("1", "1", "0"), ("1", "0", "1"), ("1", "0", "0"),
                              ("0", "1", "1")):
        env = dict(os.environ, FHE_FUSE_INNER_FINISH=fin, FHE_HMULT_TENS=tens,
                   FHE_FIN_STAGED=staged, PYTHONPATH=root)
        out = subprocess.run([sys.executable, "-c", code], env=env, cwd=root, capture_output=True,
                             text=True, timeout=900)
        assert out.returncode == 0, out.stderr[-2000:]
        digests.add(out.stdout.strip().splitlines()[-1])
    assert len(digests) == 1, digests


def test_tensor_core_bconv_equals_fp64_bconv():
    """The tcgen05 base conversion (csrc/bconv_umma.cuh, the default), the
    mma.sync conversions (csrc/bconv_imma.cuh) and the FP64-pipe conversion
    give the same words for HMult+Relin (batch 3, ragged last digit) and
    rotate."""
    import json
    import os
    import subprocess
    import sys

    script = os.path.join(os.path.dirname(os.path.abspath(__file__)), "helpers", "bconv_paths.py")
    res = {}
    # tcgen05 (TMEM accumulators, the default), mma.sync (register epilogue),
    # mma.sync (shared-memory transpose epilogue), FP64 pipe
    for tag, env in (("umma", {}), ("imma2", {"FHE_BCONV_UMMA": "0"}),
                     ("imma1", {"FHE_BCONV_UMMA": "0", "FHE_BCONV_LAYOUT": "1"}),
                     ("fp64", {"FHE_BCONV_IMMA": "0"})):
        r = subprocess.run([sys.executable, script], capture_output=True, text=True, timeout=600,
                           env=dict(os.environ, **env))
        assert r.returncode == 0, r.stderr[-2000:]
        res[tag] = json.loads(r.stdout.strip().splitlines()[-1])
    for tag in ("imma2", "imma1", "fp64"):
        assert res["umma"]["hmult"] == res[tag]["hmult"], tag
        assert res["umma"]["rotate"] == res[tag]["rotate"], tag


@pytest.mark.parametrize("shape", ["12,4,3", "32,16,2"])
def test_tcgen05_bconv_k_steps(shape):
    """The tcgen05 conversion at 1 and 4 K-steps (digits / P of 4 and 16
    limbs: 28 and 112 bytes of K) gives the FP64 conversion's words."""
    import json
    import os
    import subprocess
    import sys

    script = os.path.join(os.path.dirname(os.path.abspath(__file__)), "helpers", "bconv_paths.py")
    res = {}
    for tag, env in (("umma", {}), ("fp64", {"FHE_BCONV_IMMA": "0"})):
        r = subprocess.run([sys.executable, script], capture_output=True, text=True, timeout=900,
                           env=dict(os.environ, BCONV_SHAPE=shape, **env))
        assert r.returncode == 0, r.stderr[-2000:]
        res[tag] = json.loads(r.stdout.strip().splitlines()[-1])
    assert res["umma"]["hmult"] == res["fp64"]["hmult"]
    assert res["umma"]["rotate"] == res["fp64"]["rotate"]
