"""The N = 2^12 row-per-cluster NTT (csrc/ntt_row_cluster.cuh, the default
for launches of up to 5 rows per SM) is bit-identical to the C oracle
restatement of the reference transform (coremath/_kernels.py:35-99) and is
the path that ran; above the row cap the whole-row tiles run instead."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("bits,L,rows", [(36, 1, 1), (45, 13, 13), (49, 13, 26), (50, 7, 169),
                                         (45, 13, 445), (50, 40, 600), (45, 13, 741)])
def test_row_cluster_ntt_matches_oracle(bits, L, rows):
    from oracle import fast
    from paper_2503_22227_b200 import _native
    from paper_2503_22227_b200.coremath.ntt import DeviceChain
    from paper_2503_22227_b200.coremath.primes import gen_ntt_prime_chain

    n = 1 << 12
    primes = [m.value for m in gen_ntt_prime_chain(bits, n, L)]
    rng = np.random.default_rng(bits * 1000 + rows)
    midx = np.arange(rows) % L
    q = np.array(primes, dtype=np.uint64)[midx]
    a = (rng.integers(0, 1 << 62, (rows, n), dtype=np.uint64) % q[:, None]).astype(np.uint64)
    ch = DeviceChain(primes, 12)
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    for inverse in (False, True):
        buf = torch.from_numpy(a.view(np.int64)).cuda()
        c0 = _native.ntt_path_counts()["cluster"]
        ch.transform(buf, rows, inverse, limbs=L, offset=0)
        torch.cuda.synchronize()
        took = _native.ntt_path_counts()["cluster"] - c0
        assert took == (1 if rows <= 5 * sms else 0), (rows, took)
        want = fast.ntt_forward(a, primes, midx, inverse=inverse)
        got = buf.cpu().numpy().view(np.uint64)
        bad = int((got != want).any(axis=1).sum())
        assert bad == 0, (bits, L, rows, inverse, bad)


def test_row_cluster_ntt_limb_map_equals_row_tiles():
    """Rows mapped to primes through limbs and an offset (row r -> prime
    offset + r % limbs), in place: the cluster result is the same words as
    the whole-row tiles' (FHE_NTT_ROW_CLUSTER=0)."""
    import os
    import subprocess
    import sys

    code = r'''
import hashlib, numpy as np, torch
from paper_2503_22227_b200.coremath.ntt import DeviceChain
from paper_2503_22227_b200.coremath.primes import gen_ntt_prime_chain
n = 1 << 12
primes = [m.value for m in gen_ntt_prime_chain(45, n, 13)]
ch = DeviceChain(primes, 12)
g = torch.Generator(device="cuda").manual_seed(3)
y = torch.randint(0, 1 << 44, (78, n), dtype=torch.int64, device="cuda", generator=g)
ch.transform(y[:33], 33, False, limbs=11, offset=2)
ch.transform(y[33:], 45, True, limbs=5, offset=7)
ch.transform(y, 78, False, limbs=13, offset=0)
print(hashlib.sha256(y.cpu().numpy().tobytes()).hexdigest())
'''
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    digests = set()
    for flag in ("1", "0"):
        env = dict(os.environ, FHE_NTT_ROW_CLUSTER=flag, PYTHONPATH=root)
        r = subprocess.run([sys.executable, "-c", code], env=env, cwd=root, capture_output=True,
                           text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        digests.add(r.stdout.strip().splitlines()[-1])
    assert len(digests) == 1, digests
