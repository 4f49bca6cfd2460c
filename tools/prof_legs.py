"""Profiling driver (run under ncu, one GPU): one config-4 rotate step and
one rescale step at batch B (PROF_BATCH), after warm-up, inside NVTX ranges
"rotate" / "rescale".  Not a benchmark."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402

B = int(os.environ.get("PROF_BATCH", "16"))


def main():
    from paper_2503_22227_b200 import _native
    from paper_2503_22227_b200.coremath.sampling import Rng
    from paper_2503_22227_b200.keys import galois_keygen, key_switch_into

    torch.cuda.set_device(0)
    w = bench.build_workload(B)
    ctx, lib = w["ctx"], _native.lib()
    L, n = bench.LEVELS, ctx.n
    gks = galois_keygen(ctx, w["sk"], [1], Rng((45).to_bytes(32, "little")))
    elt = ctx.galois_elt_for_step(1)
    ksk = gks.for_elt(elt)
    X = w["X"]
    P, R = torch.empty_like(X), torch.empty_like(X)
    S = torch.empty((B, 2, L - 1, n), dtype=torch.int64, device="cuda")
    ws_bytes = lib.fhe_rescale_workspace(ctx.handle, 2 * B, L)
    ws = ctx.workspace(ws_bytes, "rescale")

    def rot():
        _native.check(lib.fhe_automorph(P.data_ptr(), X.data_ptr(), B * 2 * L, ctx.log_n, elt,
                                        _native.stream_handle()), "fhe_automorph")
        key_switch_into(ctx, L, P[:, 1], ksk, R[:, 0], R[:, 1], add0=P[:, 0], batch=B,
                        d_stride=2 * L * n, add_stride=2 * L * n, out_stride=2 * L * n)

    def resc():
        _native.check(lib.fhe_rescale(ctx.handle, S.data_ptr(), X.data_ptr(), 2 * B, L, 0,
                                      ws.data_ptr(), ws_bytes, _native.stream_handle()),
                      "fhe_rescale")

    for _ in range(2):
        rot()
        resc()
    torch.cuda.synchronize()
    for name, fn in (("rotate", rot), ("rescale", resc)):
        torch.cuda.nvtx.range_push(name)
        fn()
        torch.cuda.nvtx.range_pop()
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
