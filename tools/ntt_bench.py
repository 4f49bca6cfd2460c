"""NTT microbenchmark (config-2 largest shape by default): prints GB/s."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2503_22227_b200.coremath.ntt import DeviceChain  # noqa: E402
from paper_2503_22227_b200.coremath.primes import gen_ntt_prime_chain  # noqa: E402


def run(log_n=16, L=40, cts=64, bits=50, reps=5):
    n = 1 << log_n
    rows = cts * 2 * L
    primes = [m.value for m in gen_ntt_prime_chain(bits, n, L)]
    ch = DeviceChain(primes, log_n)
    buf = torch.randint(0, 1 << (bits - 1), (rows, n), dtype=torch.int64, device="cuda")
    out = []
    for inv in (False, True):
        for _ in range(2):
            ch.transform(buf, rows, inv, limbs=L, offset=0)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(reps):
            ch.transform(buf, rows, inv, limbs=L, offset=0)
        e.record()
        e.synchronize()
        ms = s.elapsed_time(e) / reps
        out.append((ms, 2 * rows * n * 8 / ms / 1e6))
    tag = os.environ.get("FHE_SM100_LIB", "default").split("/")[-1]
    print(f"{tag} logN={log_n} L={L} rows={rows} bits={bits} fwd {out[0][0]:.3f} ms {out[0][1]:.0f} GB/s"
          f" | inv {out[1][0]:.3f} ms {out[1][1]:.0f} GB/s")


if __name__ == "__main__":
    args = [int(a) for a in sys.argv[1:]]
    run(*args)
