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
compute) instead of their sum.  Inputs land in one of two persistent staging
sets (alternating per call), so the H2D copies of a call overlap the tail of
the previous call; pool blocks (the results) are reused only after their D2H
copies finished, because the caller's stream waits for ``d2h`` before
returning.
"""

from __future__ import annotations

from dataclasses import dataclass, field

from .rnspoly import CData, Domain


@dataclass
class CopyStreams:
    """The two copy streams of a host pipeline (one per PCIe direction), and
    optionally two persistent staging sets for the inputs.

    With staging, the inputs of a call land in staging set (call % 2); the
    H2D copies of call c only wait for the compute of call c - 2 (the last
    reader of that set), so they overlap the compute and D2H tail of call
    c - 1 instead of waiting for all earlier work."""

    h2d: object
    d2h: object
    staging: list = field(default_factory=list)   # [(tensor X, tensor Y, Event read_done)]
    calls: int = 0

    @classmethod
    def create(cls) -> "CopyStreams":
        import torch

        return cls(torch.cuda.Stream(), torch.cuda.Stream())

    def staging_set(self, shape):
        """(X, Y, event) of this call's staging set, allocated on first use."""
        import torch

        if len(self.staging) < 2 or tuple(self.staging[0][0].shape) != tuple(shape):
            self.staging = [(torch.empty(shape, dtype=torch.int64, device="cuda"),
                             torch.empty(shape, dtype=torch.int64, device="cuda"), None)
                            for _ in range(2)]
        return self.calls % 2


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
    slot = streams.staging_set(tuple(host_x.shape))
    X, Y, read_done = streams.staging[slot]
    # the staging set's last reader is the compute of two calls ago
    if read_done is not None:
        streams.h2d.wait_event(read_done)
    staged = []
    for b in range(batch):
        with torch.cuda.stream(streams.h2d):
            X[b].copy_(host_x[b], non_blocking=True)
            Y[b].copy_(host_y[b], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(streams.h2d)
        staged.append((CData.wrap(X[b].reshape(-1), 2, level, n, Domain.EVALUATION),
                       CData.wrap(Y[b].reshape(-1), 2, level, n, Domain.EVALUATION), ev))
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
    done_all = torch.cuda.Event()
    done_all.record(comp)
    streams.staging[slot] = (X, Y, done_all)
    streams.calls += 1
    # result blocks return to the pool only after their D2H copies
    comp.wait_stream(streams.d2h)
    return results
