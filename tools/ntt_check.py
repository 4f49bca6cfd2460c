"""Debug helper: device NTT vs the C oracle over (log_n, bits) combinations."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from oracle import fast  # noqa: E402
from paper_2503_22227_b200.coremath.ntt import NttChain  # noqa: E402
from paper_2503_22227_b200.coremath.primes import gen_ntt_prime_chain  # noqa: E402

for log_n in [int(v) for v in os.environ.get("LOGNS", "4 6 8 9 10 11 12 13 14 16").split()]:
    for bits in (36, 45, 49, 50, 55):
        n = 1 << log_n
        L = 2
        primes = [m.value for m in gen_ntt_prime_chain(bits, n, L)]
        rng = np.random.default_rng(log_n * 100 + bits)
        a = np.stack([rng.integers(0, primes[r % L], n, dtype=np.uint64) for r in range(2 * L)])
        ch = NttChain(primes, n)
        f = ch.forward(a)
        i = ch.inverse(a)
        wf = fast.ntt_forward(a, primes)
        wi = fast.ntt_inverse(a, primes)
        okf, oki = (f == wf).all(), (i == wi).all()
        print(f"logN={log_n:2d} bits={bits} fwd={'ok' if okf else 'BAD'} inv={'ok' if oki else 'BAD'}"
              + ("" if okf else f" first bad idx {np.argwhere(f != wf)[0]} got {f[tuple(np.argwhere(f != wf)[0])]} want {wf[tuple(np.argwhere(f != wf)[0])]}"))
