"""Parity of the kernels behind the headline numbers, at the shapes the bench
times, against the C oracle restatement.

* Batched NTT at the config-2 sweep's largest shapes: N=2^16, 50-bit primes,
  64 ciphertexts x 2 polys x L limbs (L=40: 5120 rows, the roofline launch;
  L=5: 640 rows), forward and inverse, every row compared with
  oracle/c/fhe_oracle.c (coremath/_kernels.py:35-99 restated).  The default
  large-batch path (fhe_ntt_path_count) must be the one that ran.
* Config 4 (N=2^16, L=30, hybrid dnum=3) operators over batches of DISTINCT
  ciphertexts (the bench's batch sizes 8 and 16): fhe_hmult_relin,
  fhe_keyswitch, rotate (automorphism + key switch) and fhe_rescale, each
  batch item checked against the per-item oracle (tensor -> hybrid key
  switch -> add, galois_perm, rescale).  A row mix-up inside a residue-class
  group of the fused transforms would show here and not with identical items.
"""

import numpy as np
import pytest

from fhe_testutil import seeded_rng, to_u64

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

LARGE_PATHS = ("fused_tma", "cluster")


def _rows(primes, n, rows, seed):
    rng = np.random.default_rng(seed)
    L = len(primes)
    q = np.array(primes, dtype=np.uint64)[np.arange(rows) % L]
    # one draw per row, bounded by the row's prime (uniform residues)
    return (rng.integers(0, 1 << 62, (rows, n), dtype=np.uint64) % q[:, None]).astype(np.uint64)


def _paths():
    from paper_2503_22227_b200 import _native

    return _native.ntt_path_counts()


def _large_path_delta(before, after):
    return sum(after[k] - before[k] for k in LARGE_PATHS)


@pytest.mark.parametrize("L", [5, 40], ids=["640rows", "5120rows"])
def test_config2_ntt_full_shape_matches_oracle(L):
    import torch

    from oracle import fast
    from paper_2503_22227_b200.coremath.ntt import DeviceChain
    from paper_2503_22227_b200.coremath.primes import gen_ntt_prime_chain

    log_n, n = 16, 1 << 16
    rows = 64 * 2 * L
    primes = [m.value for m in gen_ntt_prime_chain(50, n, L)]
    a = _rows(primes, n, rows, 20261017 + L)
    ch = DeviceChain(primes, log_n)
    dev = torch.from_numpy(a.view(np.int64)).cuda()
    midx = np.arange(rows) % L
    for inverse in (False, True):
        buf = dev.clone()
        p0 = _paths()
        ch.transform(buf, rows, inverse, limbs=L, offset=0)
        torch.cuda.synchronize()
        assert _large_path_delta(p0, _paths()) == 1, (_paths(), "large-batch path not taken")
        step = 256
        for r0 in range(0, rows, step):
            want = fast.ntt_forward(a[r0:r0 + step], primes, midx[r0:r0 + step], inverse=inverse)
            got = to_u64(buf[r0:r0 + step])
            bad = np.nonzero((got != want).any(axis=1))[0]
            assert bad.size == 0, f"inverse={inverse}: rows {(bad + r0)[:8].tolist()} differ"
        del buf


@pytest.fixture(scope="module")
def c4():
    from paper_2503_22227_b200.context import Context, PoolConfig, hybrid_params
    from paper_2503_22227_b200.keys import galois_keygen, keygen, relin_keygen

    params = hybrid_params(1 << 16, 30, bits=50, special=10, special_bits=50, dnum=3,
                           scale=float(2 ** 49))
    ctx = Context(params, PoolConfig(unit_mb=200, cap_mb=4096))
    sk = keygen(ctx, seeded_rng(4))
    return {"ctx": ctx, "rlk": relin_keygen(ctx, sk, seeded_rng(42)),
            "gks": galois_keygen(ctx, sk, [1], seeded_rng(45))}


def _batch(ctx, B, seed, level=30):
    """B distinct (2, level, n) evaluation-domain ciphertexts (uniform residues)."""
    Q = ctx.q_values[:level]
    rng = np.random.default_rng(seed)
    q = np.array(Q, dtype=np.uint64)[None, None, :, None]
    return (rng.integers(0, 1 << 62, (B, 2, level, ctx.n), dtype=np.uint64) % q).astype(np.uint64)


def _keys(ctx, ksk):
    return ksk.data.to_numpy().reshape(3, 2, 40, ctx.n)


@pytest.mark.parametrize("B", [8, 16])
def test_batched_hmult_relin_distinct_items_vs_oracle(c4, B):
    import torch

    from oracle import fast
    from paper_2503_22227_b200.keys import hmult_relin_into

    ctx, rlk = c4["ctx"], c4["rlk"]
    Q, P = ctx.q_values, ctx.special_values
    x, y = _batch(ctx, B, 100 + B), _batch(ctx, B, 200 + B)
    X = torch.from_numpy(x.view(np.int64)).cuda()
    Y = torch.from_numpy(y.view(np.int64)).cuda()
    out = torch.empty_like(X)
    p0 = _paths()
    hmult_relin_into(ctx, 30, X, Y, rlk, out[:, 0], out[:, 1], batch=B)
    torch.cuda.synchronize()
    assert _large_path_delta(p0, _paths()) >= 1, "key switch transforms missed the large path"
    keys = _keys(ctx, rlk)
    got = to_u64(out)
    for b in range(B):
        d0, d1, d2 = fast.tensor(x[b], y[b], Q)
        kb, ka = fast.key_switch(d2, keys, Q, alpha=ctx.ks_alpha, special=P)
        assert np.array_equal(got[b, 0], fast.add(d0, kb, Q)), f"item {b} poly 0"
        assert np.array_equal(got[b, 1], fast.add(d1, ka, Q)), f"item {b} poly 1"


def test_batched_keyswitch_and_rotate_distinct_items_vs_oracle(c4):
    import torch

    from oracle import fast
    from oracle import rns_oracle as orc
    from paper_2503_22227_b200 import _native
    from paper_2503_22227_b200.keys import key_switch_into

    ctx, gks = c4["ctx"], c4["gks"]
    Q, P = ctx.q_values, ctx.special_values
    B, L, n = 8, 30, ctx.n
    elt = ctx.galois_elt_for_step(1)
    ksk = gks.for_elt(elt)
    c = _batch(ctx, B, 300)
    C = torch.from_numpy(c.view(np.int64)).cuda()
    # plain batched key switch of poly 1, added to poly 0
    K = torch.empty_like(C)
    key_switch_into(ctx, L, C[:, 1], ksk, K[:, 0], K[:, 1], add0=C[:, 0], batch=B,
                    d_stride=2 * L * n, add_stride=2 * L * n, out_stride=2 * L * n)
    # rotate: automorphism of both polys, then the key switch (ckks.py:413-433)
    Pm = torch.empty_like(C)
    R = torch.empty_like(C)
    lib = _native.lib()
    _native.check(lib.fhe_automorph(Pm.data_ptr(), C.data_ptr(), B * 2 * L, ctx.log_n, elt,
                                    _native.stream_handle()), "fhe_automorph")
    key_switch_into(ctx, L, Pm[:, 1], ksk, R[:, 0], R[:, 1], add0=Pm[:, 0], batch=B,
                    d_stride=2 * L * n, add_stride=2 * L * n, out_stride=2 * L * n)
    torch.cuda.synchronize()
    keys = _keys(ctx, ksk)
    perm = orc.galois_perm(n, elt)
    gk, gr = to_u64(K), to_u64(R)
    for b in range(B):
        kb, ka = fast.key_switch(c[b, 1], keys, Q, alpha=ctx.ks_alpha, special=P)
        assert np.array_equal(gk[b, 0], fast.add(c[b, 0], kb, Q)), f"keyswitch item {b}"
        assert np.array_equal(gk[b, 1], ka), f"keyswitch item {b} poly 1"
        pc = c[b][:, :, perm]
        kb, ka = fast.key_switch(pc[1], keys, Q, alpha=ctx.ks_alpha, special=P)
        assert np.array_equal(gr[b, 0], fast.add(pc[0], kb, Q)), f"rotate item {b}"
        assert np.array_equal(gr[b, 1], ka), f"rotate item {b} poly 1"


def test_batched_rescale_distinct_items_vs_oracle(c4):
    import torch

    from oracle import fast
    from paper_2503_22227_b200 import _native

    ctx = c4["ctx"]
    Q = ctx.q_values
    B, L, n = 16, 30, ctx.n
    c = _batch(ctx, B, 400)
    C = torch.from_numpy(c.view(np.int64)).cuda()
    S = torch.empty((B, 2, L - 1, n), dtype=torch.int64, device="cuda")
    lib = _native.lib()
    ws_bytes = lib.fhe_rescale_workspace(ctx.handle, 2 * B, L)
    ws = ctx.workspace(ws_bytes, "rescale")
    _native.check(lib.fhe_rescale(ctx.handle, S.data_ptr(), C.data_ptr(), 2 * B, L, 0,
                                  ws.data_ptr(), ws_bytes, _native.stream_handle()), "fhe_rescale")
    torch.cuda.synchronize()
    got = to_u64(S)
    for b in range(B):
        assert np.array_equal(got[b], fast.rescale(c[b], Q[:L])), f"rescale item {b}"


def test_hmult_relin_output_aliasing_input(c4):
    """fhe_sm100.h allows out0/out1 to alias x's polys: the in-place result
    equals the out-of-place one (batch 8, distinct items)."""
    import torch

    from paper_2503_22227_b200.keys import hmult_relin_into

    ctx, rlk = c4["ctx"], c4["rlk"]
    B = 8
    X = torch.from_numpy(_batch(ctx, B, 500).view(np.int64)).cuda()
    Y = torch.from_numpy(_batch(ctx, B, 600).view(np.int64)).cuda()
    out = torch.empty_like(X)
    hmult_relin_into(ctx, 30, X, Y, rlk, out[:, 0], out[:, 1], batch=B)
    hmult_relin_into(ctx, 30, X, Y, rlk, X[:, 0], X[:, 1], batch=B)
    torch.cuda.synchronize()
    assert torch.equal(X, out)
