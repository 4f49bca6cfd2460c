"""Lockstep evaluation of independent query units as one batch.

The digit units of a comparison (pdq/compare.py `digit_unit`) run the same
sequence of evaluator calls on different ciphertexts; only some constants
(the LT scaling p^-(k-1-j)) differ per unit.  `BatchEval` runs that sequence
once over a contiguous (B, polys, level, N) block:

* tensor products and key switches are single batched launches
  (`fhe_tensor(batch=B)`, `fhe_keyswitch(batch=B)`), rescales one
  `fhe_rescale` over 2B polys;
* additions are single element-wise launches over the whole block;
* constants enter as per-unit plaintexts stacked to the block's shape.

Every kernel is the one the per-unit path uses, applied to the same words,
so the unstacked results are bit-identical to running the units one by one
(CkksEval, evaluator.py:54-188) -- tests/test_gpu_pdq.py checks the query
results against the reference's own run.
"""

from __future__ import annotations

import numpy as np

from .. import _native
from ..keys import key_switch_into
from ..rnspoly import CData, Domain
from ..schemes.ckks import (
    CkksCiphertext,
    ScaleMismatch,
    scalar_plaintext,
)
from .evaluator import RETAG_RTOL, CkksEval


class CtBatch:
    """B ciphertexts of 2 polys at one level and one scale."""

    def __init__(self, data: CData, count: int, level: int, scale: float):
        self.data = data
        self.count = count
        self.level = level
        self.scale = scale

    def view(self):
        n = self.data.n
        return self.data._buf[: self.count * 2 * self.level * n].view(self.count, 2, self.level, n)


class BatchEval:
    """CkksEval's arithmetic over CtBatch blocks (same level/scale rules)."""

    def __init__(self, ev: CkksEval):
        self.ev = ev
        self.ctx = ev.ctx

    # -- packing --------------------------------------------------------------------------
    def _new(self, count: int, polys: int, level: int) -> CData:
        return CData(self.ctx.pool, count * polys, level, self.ctx.n, Domain.EVALUATION,
                     zero=False)

    def stack(self, cts: list) -> CtBatch:
        lv, sc = cts[0].level, cts[0].scale
        if any(c.level != lv or c.scale != sc or c.data.size_poly != 2 for c in cts):
            raise ValueError("lockstep batch needs equal levels, scales and 2 components")
        out = CtBatch(self._new(len(cts), 2, lv), len(cts), lv, sc)
        v = out.view()
        for i, c in enumerate(cts):
            v[i].copy_(c.data.view())
        return out

    def unstack(self, b: CtBatch) -> list:
        v = b.view()
        outs = []
        for i in range(b.count):
            cd = CData(self.ctx.pool, 2, b.level, self.ctx.n, Domain.EVALUATION, zero=False)
            cd.view().copy_(v[i])
            outs.append(CkksCiphertext(cd, b.scale, b.level))
        return outs

    # -- primitives -----------------------------------------------------------------------
    def _q_last(self, level: int) -> float:
        return float(self.ctx.q_values[level - 1])

    def _rescale(self, b: CtBatch, scale: float) -> CtBatch:
        lib = _native.lib()
        polys = 2 * b.count
        out = CtBatch(self._new(b.count, 2, b.level - 1), b.count, b.level - 1, scale)
        ws_bytes = lib.fhe_rescale_workspace(self.ctx.handle, polys, b.level)
        ws = self.ctx.workspace(ws_bytes, "rescale")
        _native.check(lib.fhe_rescale(self.ctx.handle, out.data._buf.data_ptr(),
                                      b.data._buf.data_ptr(), polys, b.level, 0, ws.data_ptr(),
                                      ws_bytes, _native.stream_handle()), "fhe_rescale")
        return out

    def _ew(self, op, out, a, bb, rows: int, level: int):
        """Element-wise op over a contiguous block: row r is limb r % level."""
        from ..rnspoly import ew

        ew(self.ctx.chain, op, out, a, bb, None, rows=rows, limbs=level)

    def _const_block(self, kind: str, values, level: int, scale: float, both: bool, key):
        """(B, 2, level, N) block of per-unit plaintexts: [pt_i, pt_i] (both)
        or [pt_i, 0].  Blocks are read-only inputs of the element-wise ops and
        every query uses the same constants, so they are kept in the
        context's plaintext LRU (schemes/ckks.py PlaintextCache)."""
        from ..schemes.ckks import plaintext_cache

        def make():
            import torch

            n = self.ctx.n
            blk = torch.zeros((len(values), 2, level, n), dtype=torch.int64, device="cuda")
            for i, z in enumerate(values):
                pt = key(z, level, scale)
                blk[i, 0].copy_(pt.data.view()[0])
                if both:
                    blk[i, 1].copy_(pt.data.view()[0])
            return blk

        ck = ("block", kind, tuple(complex(v) for v in values), level, float(scale), both)
        return plaintext_cache(self.ctx).get(ck, make)

    def _mul_scalar_raw(self, b: CtBatch, zs, scale: float) -> CtBatch:
        """ckks_multiply_scalar per unit (plaintext Re z + Im z X^(n/2) at
        `scale`), keeping the product scale b.scale * scale."""
        out = CtBatch(self._new(b.count, 2, b.level), b.count, b.level, b.scale * scale)
        blk = self._const_block("scalar", zs, b.level, scale, True,
                                lambda z, lv, s: scalar_plaintext(self.ctx, complex(z), s, lv))
        self._ew(_native.EW_MUL, out.data._buf, b.data._buf, blk, b.count * 2 * b.level, b.level)
        return out

    # -- CkksEval operations ----------------------------------------------------------------
    def drop(self, b: CtBatch, level: int) -> CtBatch:
        while b.level > level:
            s = b.scale
            b = self._rescale(self._mul_scalar_raw(b, [1.0] * b.count, self._q_last(b.level)), s)
        return b

    def _pairwise(self, a: CtBatch, b: CtBatch):
        lv = min(a.level, b.level)
        return self.drop(a, lv), self.drop(b, lv)

    def _retag(self, a: CtBatch, b: CtBatch) -> CtBatch:
        if a.scale == b.scale:
            return b
        if abs(a.scale - b.scale) > RETAG_RTOL * a.scale:
            raise ScaleMismatch(f"scales {a.scale} and {b.scale} too far apart to retag")
        return CtBatch(b.data, b.count, b.level, a.scale)

    def add(self, a: CtBatch, b: CtBatch) -> CtBatch:
        a, b = self._pairwise(a, b)
        b = self._retag(a, b)
        out = CtBatch(self._new(a.count, 2, a.level), a.count, a.level, a.scale)
        self._ew(_native.EW_ADD, out.data._buf, a.data._buf, b.data._buf,
                 a.count * 2 * a.level, a.level)
        return out

    def add_many(self, bs: list) -> CtBatch:
        acc = bs[0]
        for b in bs[1:]:
            acc = self.add(acc, b)
        return acc

    def add_const(self, b: CtBatch, cs) -> CtBatch:
        """Per-unit constants cs (or one constant for all)."""
        cs = list(cs) if np.ndim(cs) else [cs] * b.count
        ev = self.ev

        def pt(c, lv, s):
            return ev._encode_cached(("const", complex(c)),
                                     np.full(ev.slots, c, dtype=np.complex128), lv, s)

        blk = self._const_block("const", cs, b.level, b.scale, False, pt)
        out = CtBatch(self._new(b.count, 2, b.level), b.count, b.level, b.scale)
        self._ew(_native.EW_ADD, out.data._buf, b.data._buf, blk, b.count * 2 * b.level, b.level)
        return out

    def _relin_rescale(self, t3: CData, count: int, level: int, scale: float) -> CtBatch:
        n = self.ctx.n
        v3 = t3._buf[: count * 3 * level * n].view(count, 3, level, n)
        lin = CtBatch(self._new(count, 2, level), count, level, scale)
        o = lin.view()
        key_switch_into(self.ctx, level, v3[:, 2], self.ev.relin_key, o[:, 0], o[:, 1],
                        add0=v3[:, 0], add1=v3[:, 1], batch=count, d_stride=3 * level * n,
                        add_stride=3 * level * n, out_stride=2 * level * n)
        return self._rescale(lin, scale / self._q_last(level))

    def _tensor(self, a: CtBatch, b: CtBatch | None) -> CData:
        lib = _native.lib()
        n, lv = self.ctx.n, a.level
        t3 = self._new(a.count, 3, lv)
        _native.check(lib.fhe_tensor(self.ctx.chain.handle, t3._buf.data_ptr(),
                                     a.data._buf.data_ptr(),
                                     None if b is None else b.data._buf.data_ptr(), lv, a.count,
                                     2 * lv * n, 2 * lv * n, 3 * lv * n, 1 if b is None else 0,
                                     _native.stream_handle()), "fhe_tensor")
        return t3

    def mul(self, a: CtBatch, b: CtBatch) -> CtBatch:
        for _ in range(a.count):
            self.ev._count("mul")
        a, b = self._pairwise(a, b)
        return self._relin_rescale(self._tensor(a, b), a.count, a.level, a.scale * b.scale)

    def square(self, a: CtBatch) -> CtBatch:
        for _ in range(a.count):
            self.ev._count("square")
        return self._relin_rescale(self._tensor(a, None), a.count, a.level, a.scale * a.scale)

    def mul_scalar(self, b: CtBatch, zs) -> CtBatch:
        zs = list(zs) if np.ndim(zs) else [zs] * b.count
        s = b.scale
        out = self._rescale(self._mul_scalar_raw(b, zs, self._q_last(b.level)), s)
        out.scale = s
        return out
