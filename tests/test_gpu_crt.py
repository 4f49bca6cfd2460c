"""Device CRT lift (csrc/crt.cu, fhe_crt_lift) against the exact Python-
integer formulas the reference evaluates (crt.py:84-100 + ckks.py:157-166,
bgv.py:89-101, bfv.py:106-117), on random residues and on the edge values
0, 1, Q-1, Q//2, Q//2+1, +-2^1023-scale magnitudes."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _ctx(L, bits, n=4096):
    import paper_2503_22227_b200.context as pctx
    from paper_2503_22227_b200.context import Context, EncryptionParams, PoolConfig, Scheme
    from paper_2503_22227_b200.coremath.primes import gen_ntt_prime_chain

    primes = tuple(m.value for m in gen_ntt_prime_chain(bits, n, L))
    old = pctx.MAX_CHAIN_LEN
    pctx.MAX_CHAIN_LEN = max(old, L)  # as the reference needs for long chains
    try:
        return Context(EncryptionParams(Scheme.BGV, n, primes, plain_modulus=65537),
                       PoolConfig(unit_mb=16, cap_mb=256)), primes
    finally:
        pctx.MAX_CHAIN_LEN = old


@pytest.mark.parametrize("L,bits", [(1, 45), (3, 45), (13, 45), (30, 50)])
def test_lift_modes_match_python_integers(L, bits):
    import torch

    from paper_2503_22227_b200 import _native
    from paper_2503_22227_b200.coremath.crt import device_lift

    ctx, primes = _ctx(L, bits)
    n = ctx.n
    Q = 1
    for q in primes:
        Q *= q
    rng = np.random.default_rng(L)
    vals = [int(x) for x in rng.integers(0, 1 << 62, n)]
    vals = [(v * 0x9E3779B97F4A7C15 ** (L + 1)) % Q for v in vals]  # spread over [0, Q)
    edge = [0, 1, Q - 1, Q // 2, Q // 2 + 1, Q // 2 - 1, (1 << 70) % Q, (Q - (1 << 90)) % Q]
    vals[:len(edge)] = edge
    # small centred values (what a decryption produces)
    for i in range(len(edge), 64):
        s = int(rng.integers(-(1 << 60), 1 << 60))
        vals[i] = s % Q
    rows = np.array([[v % q for v in vals] for q in primes], dtype=np.uint64)
    dev = torch.from_numpy(rows.view(np.int64)).cuda()
    cen = [v - Q if v > Q // 2 else v for v in vals]
    scale = 2.0 ** 40
    got = device_lift(ctx, dev, L, _native.CRT_FLOAT, scale=scale).cpu().numpy()
    want = []
    for c in cen:
        try:
            want.append(float(c) / scale)
        except OverflowError:
            want.append(np.inf if c > 0 else -np.inf)
    assert np.array_equal(got, np.array(want)), "float lift differs"
    t, inv_f = 65537, 12345
    got = device_lift(ctx, dev, L, _native.CRT_MOD_T, t=t, inv_f=inv_f).cpu().numpy()
    assert [int(x) for x in got] == [(c % t) * inv_f % t for c in cen]
    got = device_lift(ctx, dev, L, _native.CRT_BFV, t=t).cpu().numpy()
    assert [int(x) for x in got] == [((t * c + Q // 2) // Q) % t for c in cen]
