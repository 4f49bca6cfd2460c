"""Host-resident batches through the device operators.

The reference runs every operator on host arrays (the CPU package keeps
ciphertexts in numpy).  A user switching to this package with ciphertexts in
(pinned) host memory wants the copies hidden behind the arithmetic; this module
does that with three CUDA streams:

* ``h2d``: host -> HBM copies of the inputs of every item, issued up front;
* the caller's current stream: the public operators (``ckks_multiply`` then
  ``ckks_relinearize``) for item i once its inputs have landed;
* ``d2h``: HBM -> host copy of item i's result once it is computed.

PCIe runs both directions at once, so a batch costs about max(H2D, D2H,
compute) instead of their sum.  Pool blocks are never touched by two streams
at the same time: the inputs of a batch are allocated before any of its
compute is enqueued (after ``h2d`` has waited for earlier work on the
compute stream), and the caller's stream waits for ``d2h`` before returning,
so result blocks are reused only after their copies finished.
"""

from __future__ import annotations

from dataclasses import dataclass

from .rnspoly import CData, Domain


@dataclass
class CopyStreams:
    """The two copy streams of a host pipeline (one per PCIe direction)."""

    h2d: object
    d2h: object

    @classmethod
    def create(cls) -> "CopyStreams":
        import torch

        return cls(torch.cuda.Stream(), torch.cuda.Stream())


def hmult_relin_host_batch(ctx, host_x, host_y, scale_x: float, scale_y: float, level: int,
                           rlk, host_out, streams: CopyStreams | None = None):
    """HMult+Relin of B ciphertext pairs held in host memory.

    host_x, host_y: pinned int64 tensors (B, 2, level, N) of evaluation-domain
    ciphertexts at ``level``; host_out: pinned (B, 2, level, N) receiving the
    relinearized products.  Each item goes through the public
    ``ckks_multiply`` -> ``ckks_relinearize``; returns the device results
    (already copied to ``host_out`` when the caller's stream reaches them)."""
    import torch

    from .schemes import ckks

    streams = streams or CopyStreams.create()
    comp = torch.cuda.current_stream()
    batch = host_x.shape[0]
    n = ctx.n
    # blocks freed by earlier work on the compute stream may be handed out below
    streams.h2d.wait_stream(comp)
    staged = []
    for b in range(batch):
        xa = CData(ctx.pool, 2, level, n, Domain.EVALUATION, zero=False)
        ya = CData(ctx.pool, 2, level, n, Domain.EVALUATION, zero=False)
        with torch.cuda.stream(streams.h2d):
            xa.view().copy_(host_x[b], non_blocking=True)
            ya.view().copy_(host_y[b], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(streams.h2d)
        staged.append((xa, ya, ev))
    results = []
    for b, (xa, ya, ev) in enumerate(staged):
        comp.wait_event(ev)
        a = ckks.CkksCiphertext(xa, scale_x, level)
        c = ckks.CkksCiphertext(ya, scale_y, level)
        r = ckks.ckks_relinearize(ctx, ckks.ckks_multiply(ctx, a, c), rlk)
        done = torch.cuda.Event()
        done.record(comp)
        streams.d2h.wait_event(done)
        with torch.cuda.stream(streams.d2h):
            host_out[b].copy_(r.data.view(), non_blocking=True)
        results.append(r)
    comp.wait_stream(streams.d2h)
    return results
