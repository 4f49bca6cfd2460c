"""CUDA-graph replay of a private-dataset query.

A query is ~300 operator calls and ~800 small kernels at N = 4096; in eager
mode the host (Python operator dispatch, 13-35 us per call) dominates the
latency.  Everything before the two-party inverse is pure device work with a
fixed shape for a given (engine, query), so it is recorded ONCE into a CUDA
graph and replayed per query with one launch:

* the device part runs once eagerly first, so every cached plaintext constant,
  workspace and table the circuit touches already lives in HBM (nothing is
  uploaded or allocated on the device while capturing);
* during capture the context's memory pool is swapped for a private arena
  that belongs to the graph: the capture's temporaries reuse each other's
  blocks exactly as they will on every replay, and no block the graph
  writes can be handed to anyone else afterwards;
* inputs are the engine's resident column ciphertexts and the query's
  constant columns (passed at capture and kept alive here); the outputs are
  the captured ciphertexts, overwritten by every replay -- a result is valid
  until the next replay of the same CapturedQuery;
* the host part (two-party inverse: mask, decrypt, reciprocal, re-encrypt)
  runs eagerly; the products after it (unmask with the same r, then one or
  two ciphertext products) are a second graph, captured at the first run:
  per run the fresh ciphertext and the mask's encoding (host FFT, as the
  reference) are copied into that graph's static inputs before its replay.

Every replay computes the same words as the eager path (same kernels, same
order); tests/test_gpu_pdq_graph.py checks them against the reference goldens.
Single-GPU only (the sharded layouts exchange through collectives).
"""

from __future__ import annotations

import numpy as np

from ..pools import MemoryPool
from ..rnspoly import CData
from ..schemes.ckks import (CkksCiphertext, CkksPlaintext, ckks_multiply_plain, ckks_rescale,
                            embed_inverse, encode_embedded)
from .engine import PdqEngine, QueryResult, QuerySpec


class CapturedQuery:
    def __init__(self, engine: PdqEngine, spec: QuerySpec, temps: dict | None = None,
                 arena_mb: int = 512, lanes: bool = True):
        import torch

        if engine.group is not None and engine.group.world > 1:
            raise ValueError("CUDA-graph capture is single-GPU (the sharded query exchanges "
                             "through collectives)")
        self.engine, self.spec, self.temps = engine, spec, temps or {}
        ctx = engine.ev.ctx
        # 1. eager warm-up of the device part (no inverse: consumes no randomness)
        engine.device_part(spec, self.temps)
        torch.cuda.synchronize()
        # 2. capture the device part with a private pool arena
        self.pool = MemoryPool(1, unit_mb=arena_mb, cap_mb=arena_mb)
        self.graph = torch.cuda.CUDAGraph()
        # lanes: the independent unit groups are captured on the context's
        # StreamPool streams (fork / join inside the capture), so the graph
        # runs them as concurrent branches.  The garbage collector is off
        # while capturing: a collected Context / DeviceChain frees its native
        # tables (cudaFree), which is illegal while a stream captures.
        import gc

        gc.collect()
        gc_was_on = gc.isenabled()
        gc.disable()
        saved, saved_lanes = ctx.pool, engine.use_lanes
        ctx.pool = self.pool
        engine.use_lanes = lanes and ctx.worker is not None
        try:
            with torch.cuda.graph(self.graph):
                self.parts = engine.device_part(spec, self.temps)
        finally:
            ctx.pool, engine.use_lanes = saved, saved_lanes
            if gc_was_on:
                gc.enable()
        torch.cuda.synchronize()

    def replay(self) -> dict:
        """The device part: one graph launch on the current stream."""
        self.graph.replay()
        return self.parts

    def run(self, channel=None, rng=None) -> QueryResult:
        parts = self.replay()
        if self.spec.agg not in ("avg", "ratio"):
            return self.engine.finish(self.spec, parts, channel, rng)
        return self._finish_inverse(parts, channel, rng)

    # -- the products after the two-party inverse ---------------------------------
    def _post(self, parts: dict, fresh: CkksCiphertext, pt: CkksPlaintext):
        """engine.finish's device work after the reciprocal (reference
        engine.py:209-244, two_party_multiply_inverse's last line)."""
        ev = self.engine.ev
        inv = ckks_rescale(ev.ctx, ckks_multiply_plain(ev.ctx, fresh, pt))
        inv.scale = fresh.scale
        if self.spec.agg == "avg":
            return {"avg": ev.mul(parts["total"], inv), "count": parts["count"]}
        return {"ratio": ev.mul(ev.mul(parts["num"], inv), parts["mask"])}

    def _staged(self, name: str, key, fn, inputs: list):
        """fn(*inputs) replayed from a graph captured at its first use (per
        name and metadata key): the first call runs eagerly, then records fn
        over static copies of the inputs (device plaintexts / ciphertexts) in a
        private pool; later calls copy the inputs in and replay."""
        import gc

        import torch

        st = self._finish_graphs.get(name)
        if st is not None and st["key"] == key:
            for buf, x in zip(st["bufs"], inputs):
                buf.copy_(x.data.view())
            st["graph"].replay()
            return st["outs"]
        result = fn(*inputs)
        ctx = self.engine.ev.ctx
        bufs, statics = [], []
        for x in inputs:
            b = x.data.view().clone()
            cd = CData.wrap(b.reshape(-1), x.data.size_poly, x.data.size_modulus, ctx.n,
                            x.data.domains[0])
            statics.append(type(x)(cd, x.scale, x.level))
            bufs.append(b)
        torch.cuda.synchronize()
        pool = MemoryPool(1, unit_mb=64, cap_mb=64)
        g = torch.cuda.CUDAGraph()
        gc.collect()
        gc_was_on = gc.isenabled()
        gc.disable()
        saved = ctx.pool
        ctx.pool = pool
        try:
            with torch.cuda.graph(g):
                outs = fn(*statics)
        finally:
            ctx.pool = saved
            if gc_was_on:
                gc.enable()
        torch.cuda.synchronize()
        self._finish_graphs[name] = {"key": key, "graph": g, "bufs": bufs, "outs": outs,
                                     "pool": pool}
        return result

    def _finish_inverse(self, parts: dict, channel, rng) -> QueryResult:
        ev, cfg = self.engine.ev, self.engine.cfg
        if not hasattr(self, "_finish_graphs"):
            self._finish_graphs = {}
        ct = parts["count"] if self.spec.agg == "avg" else parts["denom"]
        # two_party_multiply_inverse (engine.py) with its two mask products
        # replayed from graphs: the same random draws in the same order
        rng = rng or np.random.default_rng()
        e = cfg.mask_exp_range
        r = rng.uniform(2.0 ** -e, 2.0 ** e, ev.slots)
        r *= rng.choice([-1.0, 1.0], ev.slots)
        # r is encoded twice (at the masked and the fresh ciphertext's level):
        # one embedding, two scalings -- the words ev.encode gives each time
        emb = embed_inverse(r.astype(np.complex128), ev.ctx.n)
        pt1 = encode_embedded(ev.ctx, emb, ev._q_last(ct), ct.level)

        def mask(p):
            out = ckks_rescale(ev.ctx, ckks_multiply_plain(ev.ctx, ct, p))
            out.scale = ct.scale
            return out

        masked = self._staged("mask", (ct.level, ct.scale, pt1.scale), mask, [pt1])
        fresh, flags = channel.reciprocal(masked)
        pt = encode_embedded(ev.ctx, emb, ev._q_last(fresh), fresh.level)
        cts = self._staged("post", (fresh.level, fresh.scale, pt.scale),
                           lambda f, p: self._post(parts, f, p), [fresh, pt])
        return QueryResult(self.spec.agg, cts, {"recip_flags": flags.tolist()})
