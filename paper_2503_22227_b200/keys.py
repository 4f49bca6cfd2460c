"""Secret / public / relinearisation / Galois keys and the key-switch
primitive, with all polynomial arithmetic on the device.

Sampling replays the reference's host RNG call order exactly (keys.py:69-179,
sampling.py:37-52), so with the default parameters (alpha = 1, no special
primes) every key word is bit-identical to the reference's.  With special
primes P and digits of alpha primes (hybrid key switching) the key for digit
d encrypts [P]_{q_j} * payload_j on the digit's primes j and 0 elsewhere, over
the extended chain Q|P; for P = 1, alpha = 1 this is the reference's gadget
row ``_gadget_rows`` (keys.py:128-141).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _native
from .context import Context, Scheme
from .coremath.modmath import ParameterError
from .coremath.sampling import SEED_BYTES, Rng, fresh_seed, signed_to_residues
from .rnspoly import CData, Domain, cdata_new, ew


@dataclass
class SecretKey:
    coeffs: np.ndarray   # signed ternary, length n
    s: CData             # (1, L+K, n) evaluation domain, Q primes then P primes
    seed: bytes


@dataclass
class PublicKey:
    data: CData          # (2, L, n) [b, a] evaluation domain
    a_seed: bytes | None = None


class KSwitchKey:
    """dnum digit pairs stored as one contiguous (2*dnum, L+K, n) block, the
    layout fhe_keyswitch reads; ``digits`` exposes per-digit (2, L+K, n) views
    like the reference's list of CData (keys.py:43-48)."""

    def __init__(self, data: CData, dnum: int, target_elt: int | None = None):
        self.data = data
        self.dnum = dnum
        self.target_elt = target_elt

    @property
    def digits(self) -> list[CData]:
        d = self.data
        per = 2 * d.size_modulus * d.n
        return [CData.wrap(d._buf[i * per:(i + 1) * per], 2, d.size_modulus, d.n)
                for i in range(self.dnum)]


@dataclass
class GaloisKeys:
    keys: dict = field(default_factory=dict)  # elt -> KSwitchKey

    def for_elt(self, elt: int) -> KSwitchKey:
        try:
            return self.keys[elt]
        except KeyError:
            raise ParameterError(f"no galois key for element {elt}") from None


class LevelMismatch(ParameterError):
    pass


# -- device helpers --------------------------------------------------------------


def upload_rows(rows: np.ndarray):
    import torch

    return torch.from_numpy(np.ascontiguousarray(rows, dtype=np.uint64).view(np.int64)).cuda()


def ntt_rows(ctx: Context, t, limbs: int, offset: int = 0, inverse: bool = False):
    """In-place NTT of `limbs` contiguous rows at chain positions offset.."""
    rows = t.numel() // ctx.n
    ctx.chain.transform(t, rows, inverse, limbs=limbs, offset=offset)
    return t


# Ring degree from which keys and noise are sampled on the device (the same
# Philox stream as the host sampler, coremath/sampling.py *_device).  At
# N = 2^12 (the PDQ ring) a host encrypt spends 3.3 ms in numpy draws and
# residue expansion against 0.37 ms on the device (tools/pdq_finish_time.py);
# below 2^11 the host draws are cheaper than the launches.
DEVICE_SAMPLING_MIN_N = 1 << 11


def device_sampling(ctx: Context) -> bool:
    return ctx.n >= DEVICE_SAMPLING_MIN_N


def signed_eval(ctx: Context, coeffs, primes) -> object:
    """Small signed polynomial (host numpy, or an int64 device tensor from a
    device sampler) -> evaluation-domain rows over `primes` (a prefix of the
    context chain)."""
    import torch

    if isinstance(coeffs, torch.Tensor):
        t = torch.empty((len(primes), ctx.n), dtype=torch.int64, device="cuda")
        _native.check(_native.lib().fhe_signed_lift(ctx.chain.handle, t.data_ptr(),
                                                    coeffs.data_ptr(), ctx.n, len(primes), 0,
                                                    _native.stream_handle()), "fhe_signed_lift")
    else:
        t = upload_rows(signed_to_residues(coeffs, primes))
    return ntt_rows(ctx, t, len(primes))


def _chain_primes(ctx: Context, limbs: int):
    return (ctx.q_values + ctx.special_values)[:limbs]


# -- key generation ---------------------------------------------------------------


def keygen(ctx: Context, rng: Rng | None = None) -> SecretKey:
    rng = rng or Rng(fresh_seed())
    coeffs = rng.ternary(ctx.n)
    LK = ctx.L + ctx.K
    s = cdata_new(ctx.pool, 1, LK, ctx.n, Domain.EVALUATION, zero=False)
    s.view()[0].copy_(signed_eval(ctx, coeffs, _chain_primes(ctx, LK)))
    return SecretKey(coeffs=coeffs, s=s, seed=rng.seed)


def _rlwe_pair(ctx: Context, sk: SecretKey, rng: Rng, extra=None, a_rows=None,
               limbs: int | None = None) -> CData:
    """(b, a) with b = -(a s) + e (+ extra) over the first `limbs` chain
    primes (keys.py:77-113); evaluation domain."""
    limbs = limbs or ctx.L
    n = ctx.n
    primes = _chain_primes(ctx, limbs)
    dev = device_sampling(ctx) and ctx.params.scheme is not Scheme.BGV
    if a_rows is None:
        a_rows = ntt_rows(ctx, rng.uniform_residues_device(primes, n) if dev
                          else upload_rows(rng.uniform_residues(primes, n)), limbs)
    e = rng.cbd_error_device(n) if dev else rng.cbd_error(n)
    if ctx.params.scheme is Scheme.BGV:
        e = e * ctx.plain_modulus.value
    e_rows = signed_eval(ctx, e, primes)
    out = cdata_new(ctx.pool, 2, limbs, n, Domain.EVALUATION, zero=False)
    v = out.view()
    s_rows = sk.s.view()[0, :limbs]
    ch = ctx.chain
    ew(ch, _native.EW_NEG_MUL, v[0], a_rows, s_rows, rows=limbs, limbs=limbs)
    ew(ch, _native.EW_ADD, v[0], v[0], e_rows, rows=limbs, limbs=limbs)
    if extra is not None:
        ew(ch, _native.EW_ADD, v[0], v[0], extra, rows=limbs, limbs=limbs)
    v[1].copy_(a_rows)
    return out


def pk_gen(ctx: Context, sk: SecretKey, rng: Rng | None = None) -> PublicKey:
    rng = rng or Rng(fresh_seed())
    a_seed = rng.uniform_bytes(SEED_BYTES)
    ar = Rng(a_seed)
    a_rows = ntt_rows(ctx, ar.uniform_residues_device(ctx.q_arr(), ctx.n) if device_sampling(ctx)
                      else upload_rows(ar.uniform_residues(ctx.q_arr(), ctx.n)), ctx.L)
    return PublicKey(data=_rlwe_pair(ctx, sk, rng, a_rows=a_rows, limbs=ctx.L), a_seed=a_seed)


def _ksk_for_payload(ctx: Context, sk: SecretKey, payload, rng: Rng,
                     target_elt: int | None = None) -> KSwitchKey:
    import torch

    LK, n, D, A = ctx.L + ctx.K, ctx.n, ctx.ks_digits, ctx.ks_alpha
    data = cdata_new(ctx.pool, 2 * D, LK, n, Domain.EVALUATION, zero=False)
    for d in range(D):
        s0, na = d * A, min(A, ctx.L - d * A)
        extra = torch.zeros((LK, n), dtype=torch.int64, device="cuda")
        # [P]_{q_j} * payload_j on the digit's primes (payload itself when P = 1)
        ew(ctx.chain, _native.EW_MUL, extra[s0:s0 + na], payload[s0:s0 + na], ctx._p_mod_q,
           rows=na, limbs=na, offset=s0, b_mode=_native.B_CONST)
        pair = _rlwe_pair(ctx, sk, rng, extra=extra, limbs=LK)
        data.view()[2 * d:2 * d + 2].copy_(pair.view())
    return KSwitchKey(data, D, target_elt)


def relin_keygen(ctx: Context, sk: SecretKey, rng: Rng | None = None) -> KSwitchKey:
    """Key switching s^2 -> s (keys.py:144-160)."""
    import torch

    rng = rng or Rng(fresh_seed())
    LK = ctx.L + ctx.K
    s = sk.s.view()[0]
    s2 = torch.empty_like(s)
    ew(ctx.chain, _native.EW_MUL, s2, s, s, rows=LK, limbs=LK)
    return _ksk_for_payload(ctx, sk, s2, rng)


def automorph_rows(ctx: Context, src, elt: int):
    import torch

    out = torch.empty_like(src)
    lib = _native.lib()
    _native.check(lib.fhe_automorph(out.data_ptr(), src.data_ptr(), src.numel() // ctx.n,
                                    ctx.log_n, elt, _native.stream_handle()), "fhe_automorph")
    return out


def galois_keygen(ctx: Context, sk: SecretKey, steps, rng: Rng | None = None,
                  include_conj: bool = False) -> GaloisKeys:
    """Keys switching sigma_g(s) -> s (keys.py:163-179)."""
    rng = rng or Rng(fresh_seed())
    elts = [ctx.galois_elt_for_step(k) for k in steps]
    if include_conj:
        elts.append(ctx.conj_elt)
    out = GaloisKeys()
    s = sk.s.view()[0]
    for elt in elts:
        if elt in out.keys:
            continue
        out.keys[elt] = _ksk_for_payload(ctx, sk, automorph_rows(ctx, s, elt), rng,
                                         target_elt=elt)
    return out


# -- key switching ------------------------------------------------------------------


def key_switch_into(ctx: Context, level: int, d, ksk: KSwitchKey, out0, out1, add0=None,
                    add1=None, batch: int = 1, d_stride: int | None = None,
                    add_stride: int | None = None, out_stride: int | None = None,
                    stream=None):
    """Device key switch: out0 = add0 + b, out1 = add1 + a (fhe_keyswitch)."""
    if level > ctx.L or level < 1:
        raise LevelMismatch(f"polynomial level {level} exceeds key level")
    lib = _native.lib()
    n = ctx.n
    ws_bytes = lib.fhe_keyswitch_workspace(ctx.handle, level, batch)
    ws = ctx.workspace(ws_bytes, "keyswitch")
    _native.check(lib.fhe_keyswitch(
        ctx.handle, level, _native.ptr(d), d_stride or level * n, ksk.data._buf.data_ptr(),
        _native.ptr(add0), _native.ptr(add1), add_stride or level * n, _native.ptr(out0),
        _native.ptr(out1), out_stride or level * n, batch, ws.data_ptr(), ws_bytes,
        _native.stream_handle(stream)),
        "fhe_keyswitch")


def hmult_relin_into(ctx: Context, level: int, x, y, rlk: KSwitchKey, out0, out1,
                     batch: int = 1, in_stride: int | None = None,
                     out_stride: int | None = None, stream=None):
    """Fused tensor product + relinearization (fhe_hmult_relin): x, y are batch
    x (2, level, n) ciphertexts in_stride words apart (y may be x); out0/out1
    receive d0 + b and d1 + a -- the words of ckks_multiply followed by
    ckks_relinearize (ckks.py:308-379)."""
    if level > ctx.L or level < 1:
        raise LevelMismatch(f"polynomial level {level} exceeds key level")
    lib = _native.lib()
    n = ctx.n
    ws_bytes = lib.fhe_hmult_relin_workspace(ctx.handle, level, batch)
    ws = ctx.workspace(ws_bytes, "hmult_relin")
    _native.check(lib.fhe_hmult_relin(
        ctx.handle, level, _native.ptr(x), _native.ptr(y), in_stride or 2 * level * n,
        rlk.data._buf.data_ptr(), _native.ptr(out0), _native.ptr(out1),
        out_stride or 2 * level * n, batch, ws.data_ptr(), ws_bytes,
        _native.stream_handle(stream)), "fhe_hmult_relin")


def key_switch(ctx: Context, rows, ksk: KSwitchKey):
    """Apply a key-switch key to an evaluation-domain (level, n) polynomial;
    returns (b_rows, a_rows) on the device (keys.py:186-237)."""
    import torch

    if isinstance(rows, np.ndarray):
        rows = upload_rows(rows)
    rows = rows.contiguous()
    level = rows.shape[0]
    if level > ctx.L:
        raise LevelMismatch(f"polynomial level {level} exceeds key level")
    b = torch.empty_like(rows)
    a = torch.empty_like(rows)
    key_switch_into(ctx, level, rows, ksk, b, a)
    return b, a
