"""Profiling driver (run under ncu on ONE GPU): a batched NTT at N=2^16 and
one config-4 HMult+Relin step, after warm-up.  Not a benchmark."""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402

B = int(os.environ.get("PROF_BATCH", "8"))
ROWS = int(os.environ.get("PROF_NTT_ROWS", "1280"))


def main():
    from paper_2503_22227_b200.coremath.ntt import DeviceChain
    from paper_2503_22227_b200.coremath.primes import gen_ntt_prime_chain

    torch.cuda.set_device(0)
    n = 1 << 16
    primes = [m.value for m in gen_ntt_prime_chain(50, n, 40)]
    ch = DeviceChain(primes, 16)
    buf = torch.randint(0, 1 << 40, (ROWS, n), dtype=torch.int64, device="cuda")
    w = bench.build_workload(B)
    for _ in range(2):
        ch.transform(buf, ROWS, False, limbs=40, offset=0)
        bench.hmult_relin_step(w, B)
    torch.cuda.synchronize()
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_push("profiled")
    ch.transform(buf, ROWS, False, limbs=40, offset=0)
    ch.transform(buf, ROWS, True, limbs=40, offset=0)
    bench.hmult_relin_step(w, B)
    torch.cuda.nvtx.range_pop()
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
