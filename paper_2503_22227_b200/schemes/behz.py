"""BEHZ full-RNS BFV tensor on the device.

Host precompute mirrors the reference's BehzConstants (schemes/behz.py:58-118):
auxiliary base B of 50-bit primes sized by the same rule, plus m_sk and
m_tilde = 2^16; every constant the kernels need is packed once into a device
block (layout documented in csrc/behz.cu).  behz_tensor (behz.py:236-270) runs
as: lift (fhe_behz_lift) -> NTT over Q|Bsk -> fused tensor (fhe_tensor) ->
INTT -> scale-and-floor back to Q (fhe_behz_floor).
"""

from __future__ import annotations

import numpy as np

from .. import _native
from ..context import Context
from ..coremath.modmath import inv_mod
from ..coremath.ntt import DeviceChain
from ..coremath.primes import gen_ntt_prime_chain
from ..rnspoly import CData, Domain, cdata_new

M_TILDE_BITS = 16
M_TILDE = 1 << M_TILDE_BITS
AUX_PRIME_BITS = 50


def _shoup(w: int, q: int) -> int:
    return (w << 64) // q


def _pairs(vals, mods):
    out = []
    for v, m in zip(vals, mods):
        v %= m
        out += [v, _shoup(v, m)]
    return out


class BehzConstants:
    def __init__(self, ctx: Context, level: int):
        import torch

        self.level = level
        base = ctx.bases[level]
        self.q_values = list(base.values)
        self.q_prod = base.product
        n = ctx.n
        t = ctx.plain_modulus.value
        need_bits = self.q_prod.bit_length() + 2 * n.bit_length() + t.bit_length() + 8
        k_aux = -(-need_bits // AUX_PRIME_BITS)
        aux = gen_ntt_prime_chain(AUX_PRIME_BITS, n, k_aux + 1,
                                  extra_exclude=set(self.q_values) | {t})
        self.b_values = [m.value for m in aux[:-1]]
        self.m_sk = aux[-1].value
        self.bsk_values = self.b_values + [self.m_sk]
        self.big_values = self.q_values + self.bsk_values
        self.L, self.S = level, len(self.bsk_values)
        self.t = t
        self.big_chain = DeviceChain(self.big_values, ctx.log_n)
        Q, punc = self.q_prod, base.punctured
        inv_punc = base.punctured_inv
        Bp = 1
        for b in self.b_values:
            Bp *= b
        punc_b = [Bp // b for b in self.b_values]
        L, S = self.L, self.S
        qv, sv = self.q_values, self.bsk_values
        # lift block
        lift = _pairs([M_TILDE * inv_punc[j] for j in range(L)], qv)
        lift += [punc[j] % m for m in sv for j in range(L)]
        lift += [punc[j] % M_TILDE for j in range(L)]
        lift += [pow(-Q, -1, M_TILDE)]
        lift += [Q % m for m in sv]
        lift += _pairs([inv_mod(M_TILDE % m, m) for m in sv], sv)
        # floor block
        fl = _pairs([t % m for m in self.big_values], self.big_values)
        fl += _pairs([inv_punc[j] for j in range(L)], qv)
        fl += [punc[j] % m for m in sv for j in range(L)]
        fl += _pairs([inv_mod(Q % m, m) for m in sv], sv)
        fl += _pairs([inv_mod(punc_b[i] % b, b) for i, b in enumerate(self.b_values)],
                     self.b_values)
        fl += [punc_b[i] % q for q in qv for i in range(len(self.b_values))]
        fl += [punc_b[i] % self.m_sk for i in range(len(self.b_values))]
        fl += _pairs([inv_mod(Bp % self.m_sk, self.m_sk)], [self.m_sk])
        fl += [Bp % q for q in qv]
        to_dev = lambda v: torch.as_tensor(  # noqa: E731
            np.array([int(x) for x in v], dtype=np.uint64).view(np.int64), device="cuda")
        self.lift_dev = to_dev(lift)
        self.floor_dev = to_dev(fl)


_behz_cache: dict = {}


def behz_constants(ctx: Context, level: int) -> BehzConstants:
    key = (id(ctx), level)
    c = _behz_cache.get(key)
    if c is None:
        c = BehzConstants(ctx, level)
        _behz_cache[key] = c
    return c


def behz_tensor(ctx: Context, consts: BehzConstants, ct_a: CData, ct_b: CData) -> CData:
    """round(t * (a tensor b) / Q) in base q for 2-component coefficient-domain
    ciphertexts; returns a (3, level, n) CData (coefficient domain)."""
    import torch

    lib = _native.lib()
    L, S, n = consts.L, consts.S, ctx.n
    big = consts.big_chain
    st = _native.stream_handle()
    square = ct_b is ct_a
    lifted = []
    for ct in ((ct_a,) if square else (ct_a, ct_b)):
        buf = torch.empty((2, L + S, n), dtype=torch.int64, device="cuda")
        _native.check(lib.fhe_behz_lift(big.handle, buf.data_ptr(), ct._buf.data_ptr(), 2, L, S,
                                        consts.lift_dev.data_ptr(), st), "fhe_behz_lift")
        big.transform(buf, 2 * (L + S), False, limbs=L + S, offset=0)
        lifted.append(buf)
    prod = torch.empty((3, L + S, n), dtype=torch.int64, device="cuda")
    _native.check(lib.fhe_tensor(big.handle, prod.data_ptr(), lifted[0].data_ptr(),
                                 None if square else lifted[1].data_ptr(), L + S, 1, 0, 0, 0,
                                 1 if square else 0, st), "fhe_tensor")
    big.transform(prod, 3 * (L + S), True, limbs=L + S, offset=0)
    out = cdata_new(ctx.pool, 3, L, n, Domain.COEFFICIENT, zero=False)
    _native.check(lib.fhe_behz_floor(big.handle, out._buf.data_ptr(), prod.data_ptr(), 3, L, S,
                                     consts.floor_dev.data_ptr(), st), "fhe_behz_floor")
    return out
