"""Experiment timer (one GPU): per-launch time of small N=2^12 transforms
(the PDQ shape: 13 x 45-bit primes), back to back on one stream and as a
captured CUDA graph of the same launches, warm L2.  Not a benchmark."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402


def main():
    from paper_2503_22227_b200.coremath.ntt import DeviceChain
    from paper_2503_22227_b200.coremath.primes import gen_ntt_prime_chain

    torch.cuda.set_device(0)
    n = 1 << 12
    primes = [m.value for m in gen_ntt_prime_chain(45, n, 13)]
    ch = DeviceChain(primes, 12)
    reps = 200
    import hashlib
    g0 = torch.Generator(device="cuda").manual_seed(5)
    x = torch.randint(0, 1 << 40, (26, n), dtype=torch.int64, device="cuda", generator=g0)
    y = x.clone()
    ch.transform(y, 26, False, limbs=13, offset=0)
    z = y.clone()
    ch.transform(z, 26, True, limbs=13, offset=0)
    assert torch.equal(z, x), "round trip"
    print("fwd digest", hashlib.sha256(y.cpu().numpy().tobytes()).hexdigest()[:16])
    # graph-node floor: a trivial kernel (automorphism of one row), same harness
    from paper_2503_22227_b200 import _native
    lib = _native.lib()
    a1 = torch.randint(0, 1 << 40, (1, n), dtype=torch.int64, device="cuda")
    b1 = torch.empty_like(a1)
    triv = lambda: lib.fhe_automorph(b1.data_ptr(), a1.data_ptr(), 1, 12, 3,  # noqa: E731
                                     _native.stream_handle())
    for _ in range(5):
        triv()
    g = torch.cuda.CUDAGraph()
    st = torch.cuda.Stream()
    st.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(st):
        with torch.cuda.graph(g, stream=st):
            for _ in range(reps):
                triv()
    g.replay()
    torch.cuda.synchronize()
    s0, e0 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record()
    g.replay()
    e0.record()
    e0.synchronize()
    print(f"trivial kernel (1-row automorphism): graph {s0.elapsed_time(e0) * 1e3 / reps:6.2f} us "
          f"per launch")
    for rows in (1, 2, 13, 26, 169):
        buf = torch.randint(0, 1 << 40, (rows, n), dtype=torch.int64, device="cuda")
        out = torch.empty_like(buf)
        for inv in (False, True):
            fns = {"rows": lambda: ch.transform(buf, rows, inv, limbs=13, offset=0)}
            if os.environ.get("SMALL_NTT_MM"):
                fns["mm"] = lambda: ch.transform_mm(out, buf, rows, inv,
                                                    mod_idx=[i % 13 for i in range(rows)])
            for tag, fn in fns.items():
                for _ in range(5):
                    fn()
                torch.cuda.synchronize()
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record()
                for _ in range(reps):
                    fn()
                e.record()
                e.synchronize()
                eager = s.elapsed_time(e) * 1e3 / reps
                g = torch.cuda.CUDAGraph()
                st = torch.cuda.Stream()
                st.wait_stream(torch.cuda.current_stream())
                with torch.cuda.stream(st):
                    with torch.cuda.graph(g, stream=st):
                        for _ in range(reps):
                            fn()
                torch.cuda.synchronize()
                g.replay()
                torch.cuda.synchronize()
                s.record()
                g.replay()
                e.record()
                e.synchronize()
                graph = s.elapsed_time(e) * 1e3 / reps
                print(f"rows {rows:4d} {'inv' if inv else 'fwd'} {tag:4s}: eager {eager:6.2f} us, "
                      f"graph {graph:6.2f} us per launch")


if __name__ == "__main__":
    main()
