"""Batched NTT/INTT on the B200 vs the reference's golden vectors (config 2
sweep shapes) - bit-exact residues, checked through the C ABI."""

import numpy as np
import pytest

from fhe_testutil import digest, to_u64

pytestmark = pytest.mark.gpu


def _inputs(primes, n, rows, seed):
    rng = np.random.default_rng(seed)
    L = len(primes)
    return np.stack([rng.integers(0, primes[r % L], n, dtype=np.uint64) for r in range(rows)])


def _cases(golden):
    return [(c["key"], c) for c in golden["ntt"]]


def test_ntt_matches_reference_golden(golden, golden_arrays):
    import torch

    from paper_2503_22227_b200.coremath.ntt import DeviceChain

    arrs = golden_arrays["ntt"]
    for key, c in _cases(golden):
        primes = [int(p) for p in c["primes"]]
        n = 1 << c["log_n"]
        ch = DeviceChain(primes, c["log_n"])
        # tables: psi is the smallest primitive 2n-th root, twiddles bit-reversed
        psi, fw, iv, _ = ch.tables(0)
        assert psi == int(c["psi"][0]), key
        assert fw[:64].tolist() == arrs[key + "_psi_br"].tolist()[: min(64, n)], key
        assert iv[:64].tolist() == arrs[key + "_ipsi_br"].tolist()[: min(64, n)], key
        a = _inputs(primes, n, c["rows"], c["seed"])
        assert digest(a) == c["in_sha"]
        dev = torch.from_numpy(a.view(np.int64)).cuda()
        f = dev.clone()
        ch.transform(f, c["rows"], False, limbs=c["L"], offset=0)
        i = dev.clone()
        ch.transform(i, c["rows"], True, limbs=c["L"], offset=0)
        torch.cuda.synchronize()
        assert digest(f) == c["fwd_sha"], f"forward mismatch {key}"
        assert digest(i) == c["inv_sha"], f"inverse mismatch {key}"
        if key + "_fwd" in arrs:
            assert (to_u64(f) == arrs[key + "_fwd"]).all()


@pytest.mark.parametrize("log_n", [4, 10, 12, 13, 14, 15, 16])
def test_roundtrip_and_explicit_mod_idx(log_n):
    import torch

    from paper_2503_22227_b200.coremath.ntt import NttChain
    from paper_2503_22227_b200.coremath.primes import gen_ntt_prime_chain

    n = 1 << log_n
    primes = [m.value for m in gen_ntt_prime_chain(50, n, 4)]
    chain = NttChain(primes, n)
    rng = np.random.default_rng(log_n)
    midx = rng.integers(0, 4, 9)
    a = np.stack([rng.integers(0, primes[m], n, dtype=np.uint64) for m in midx])
    f = chain.forward(a, midx)
    back = chain.inverse(f, midx)
    assert back.tolist() == a.tolist()
    # per-row equals single-row transforms
    for r in (0, 5):
        one = NttChain([primes[midx[r]]], n).forward(a[r:r + 1], [0])
        assert one[0].tolist() == f[r].tolist()


@pytest.mark.parametrize("log_n", [12, 13, 16])
def test_extreme_inputs_match_oracle(log_n):
    """Worst cases for the lazy FP64 butterflies (values grow by up to
    0.75q per stage between reductions): rows of all q-1, alternating 0/q-1,
    all 1 and (q-1)/2, at 50-bit primes next to 2^50, forward and inverse
    against the C oracle."""
    import torch

    from oracle import fast
    from paper_2503_22227_b200.coremath.ntt import DeviceChain
    from paper_2503_22227_b200.coremath.primes import gen_ntt_prime_chain

    n = 1 << log_n
    primes = [m.value for m in gen_ntt_prime_chain(50, n, 2)]
    assert all(p > (1 << 49) for p in primes)
    rows = []
    for q in primes:
        rows += [np.full(n, q - 1, np.uint64), np.tile(np.array([0, q - 1], np.uint64), n // 2),
                 np.ones(n, np.uint64), np.full(n, (q - 1) // 2, np.uint64)]
    a = np.stack(rows)
    midx = np.repeat(np.arange(2), 4)
    ch = DeviceChain(primes, log_n)
    dev = torch.from_numpy(a.view(np.int64)).cuda()
    f = dev.clone()
    ch.transform(f, len(rows), False, mod_idx=midx)
    i = dev.clone()
    ch.transform(i, len(rows), True, mod_idx=midx)
    torch.cuda.synchronize()
    assert (to_u64(f) == fast.ntt_forward(a, primes, midx)).all()
    assert (to_u64(i) == fast.ntt_inverse(a, primes, midx)).all()


def test_fused_four_step_path_matches_oracle():
    """The opt-in fused four-step kernel (FHE_NTT_FUSED=1: one persistent
    kernel, intermediate through L2, ticketed tiles with per-group counters)
    gives the same residues; run in a child process since the switch is read
    once per process."""
    import os
    import subprocess
    import sys

    code = r'''
import numpy as np, torch
from oracle import fast
from paper_2503_22227_b200.coremath.ntt import DeviceChain
from paper_2503_22227_b200.coremath.primes import gen_ntt_prime_chain
for log_n, L, rows in ((16, 3, 21), (14, 5, 40), (13, 2, 7)):
    n = 1 << log_n
    primes = [m.value for m in gen_ntt_prime_chain(50, n, L)]
    rng = np.random.default_rng(log_n)
    a = np.stack([rng.integers(0, primes[r % L], n, dtype=np.uint64) for r in range(rows)])
    ch = DeviceChain(primes, log_n)
    dev = torch.from_numpy(a.view(np.int64)).cuda()
    f = dev.clone(); ch.transform(f, rows, False, limbs=L, offset=0)
    i = dev.clone(); ch.transform(i, rows, True, limbs=L, offset=0)
    torch.cuda.synchronize()
    midx = np.arange(rows) % L
    assert (f.cpu().numpy().view(np.uint64) == fast.ntt_forward(a, primes, midx)).all(), log_n
    assert (i.cpu().numpy().view(np.uint64) == fast.ntt_inverse(a, primes, midx)).all(), log_n
print("fused ok")
'''
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, FHE_NTT_FUSED="1", PYTHONPATH=root)
    out = subprocess.run([sys.executable, "-c", code], env=env, cwd=root, capture_output=True,
                         text=True, timeout=600)
    assert out.returncode == 0 and "fused ok" in out.stdout, out.stderr[-2000:]


def test_empty_and_partial_batches():
    """Zero rows is a no-op; a row count that is not a multiple of the limb
    count (the TMA tiles' box cannot cover a partial batch) takes the
    cp.async tiles and still matches the oracle."""
    import torch

    from oracle import fast
    from paper_2503_22227_b200.coremath.ntt import DeviceChain
    from paper_2503_22227_b200.coremath.primes import gen_ntt_prime_chain

    n, L = 1 << 16, 3
    primes = [m.value for m in gen_ntt_prime_chain(50, n, L)]
    ch = DeviceChain(primes, 16)
    buf = torch.arange(16, dtype=torch.int64, device="cuda")
    before = buf.clone()
    ch.transform(buf, 0, False, limbs=L, offset=0)
    ch.transform(buf, 0, True, limbs=L, offset=0)
    torch.cuda.synchronize()
    assert torch.equal(buf, before)
    rows = 2 * L + 1  # partial last batch of rows
    rng = np.random.default_rng(17)
    a = np.stack([rng.integers(0, primes[r % L], n, dtype=np.uint64) for r in range(rows)])
    dev = torch.from_numpy(a.view(np.int64)).cuda()
    f = dev.clone()
    ch.transform(f, rows, False, limbs=L, offset=0)
    torch.cuda.synchronize()
    assert (to_u64(f) == fast.ntt_forward(a, primes, np.arange(rows) % L)).all()
