"""CKKS over device-resident ciphertexts.

Operator surface of the reference's schemes/ckks.py:122-437 (same names,
arguments, scale bookkeeping and exceptions).  Encoding and decoding stay on
the host in float64 numpy (the canonical-embedding FFT, ckks.py:104-166) so
plaintext residues are bit-identical to the reference; everything after the
residue lift runs on the GPU:

* multiply / square  -> one fused tensor-product launch (fhe_tensor);
* relinearize/rotate -> fhe_keyswitch (ModUp, key inner product, ModDown;
                        the automorphism is a device gather);
* rescale            -> fhe_rescale (INTT of the dropped limb only, the
                        correction NTT'd back and subtracted in the
                        evaluation domain - bit-identical by linearity).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .. import _native
from ..context import Context
from ..coremath.crt import crt_centered_floats
from ..coremath.modmath import ParameterError
from ..coremath.sampling import Rng, fresh_seed, signed_to_residues
from ..keys import (KSwitchKey, PublicKey, SecretKey, automorph_rows, device_sampling,
                    hmult_relin_into,
                    key_switch_into, signed_eval, upload_rows)
from ..rnspoly import CData, Domain, cdata_new, ew

SCALE_RTOL = 1e-6


class ScaleMismatch(ParameterError):
    pass


class LevelMismatch(ParameterError):
    pass


class EncodeRangeError(ParameterError):
    pass


@dataclass
class CkksPlaintext:
    data: CData
    scale: float
    level: int


@dataclass
class CkksCiphertext:
    data: CData
    scale: float
    level: int

    def copy(self) -> "CkksCiphertext":
        return CkksCiphertext(self.data.copy(), self.scale, self.level)


# -- canonical embedding (host, float64) -------------------------------------------

def _round_half_away(x: np.ndarray) -> np.ndarray:
    return np.where(x >= 0, np.floor(x + 0.5), np.ceil(x - 0.5))


_slot_cache: dict = {}
_twist_cache: dict = {}


def _slots(n: int) -> np.ndarray:
    """k with 2k+1 = 5^j mod 2n for j < n/2 (power-of-5 slot orbit)."""
    s = _slot_cache.get(n)
    if s is None:
        s = np.empty(n // 2, dtype=np.int64)
        g = 1
        for j in range(n // 2):
            s[j] = (g - 1) // 2
            g = g * 5 % (2 * n)
        _slot_cache[n] = s
    return s


def _twist(n: int) -> np.ndarray:
    t = _twist_cache.get(n)
    if t is None:
        t = np.exp(1j * np.pi * np.arange(n) / n)
        _twist_cache[n] = t
    return t


_embed_inv_cache: dict = {}


def embed_inverse(values: np.ndarray, n: int) -> np.ndarray:
    """n/2 complex slots -> n real coefficients (the reference expression;
    the mirrored slot indices and conj(twist) are cached: same values)."""
    c = _embed_inv_cache.get(n)
    if c is None:
        idx = _slots(n)
        c = _embed_inv_cache[n] = (idx, n - 1 - idx, np.conj(_twist(n)))
    idx, ridx, ctw = c
    u = np.zeros(n, dtype=np.complex128)
    u[idx] = values
    u[ridx] = np.conj(values)
    return (np.fft.fft(u) / n * ctw).real


def embed_forward(coeffs: np.ndarray, n: int) -> np.ndarray:
    """n real coefficients -> n/2 complex slots."""
    u = np.fft.ifft(coeffs.astype(np.complex128) * _twist(n)) * n
    return u[_slots(n)]


# -- helpers -------------------------------------------------------------------------

def _new_ct(ctx: Context, polys: int, level: int) -> CData:
    return cdata_new(ctx.pool, polys, level, ctx.n, Domain.EVALUATION, zero=False)


def _poly_from_rows(ctx: Context, rows: np.ndarray, level: int) -> CData:
    """Upload host residue rows (coefficient form) and NTT them."""
    cd = cdata_new(ctx.pool, 1, level, ctx.n, Domain.EVALUATION, zero=False)
    cd.load_numpy(rows, 0)
    ctx.chain.transform(cd._buf, level, False, limbs=level, offset=0)
    return cd


def _ew(ctx: Context, op, out, a, b=None, c=None, rows=1, limbs=1, b_mode=_native.B_FULL):
    ew(ctx.chain, op, out, a, b, c, rows=rows, limbs=limbs, b_mode=b_mode)


# -- encode / decode ------------------------------------------------------------------

def ckks_encode(ctx: Context, values, scale: float | None = None,
                level: int | None = None) -> CkksPlaintext:
    n, half = ctx.n, ctx.n // 2
    level = level or ctx.L
    scale = scale or ctx.params.default_scale
    v = np.asarray(values, dtype=np.complex128).ravel()
    if v.size > half:
        raise ParameterError(f"{v.size} values exceed {half} slots")
    if v.size < half:
        v = np.concatenate([v, np.zeros(half - v.size, dtype=np.complex128)])
    return encode_embedded(ctx, embed_inverse(v, n), scale, level)


_STAGE_RING = 4


def _upload_f64(ctx: Context, host: np.ndarray):
    """float64 host vector -> device, through a small ring of pinned staging
    buffers per context (asynchronous copy; a ring slot is reused only after
    the event of its previous copy has completed)."""
    import torch

    ring = getattr(ctx, "_f64_stage", None)
    if ring is None or ring["n"] != host.size:
        ring = ctx._f64_stage = {"n": host.size, "i": 0, "slots": [
            (torch.empty(host.size, dtype=torch.float64, pin_memory=True), None)
            for _ in range(_STAGE_RING)]}
    i = ring["i"]
    ring["i"] = (i + 1) % _STAGE_RING
    buf, ev = ring["slots"][i]
    if ev is not None:
        ev.synchronize()
    buf.numpy()[:] = host
    out = torch.empty(host.size, dtype=torch.float64, device="cuda")
    out.copy_(buf, non_blocking=True)
    ev = torch.cuda.Event()
    ev.record()
    ring["slots"][i] = (buf, ev)
    return out


def encode_embedded(ctx: Context, emb: np.ndarray, scale: float, level: int) -> CkksPlaintext:
    """ckks_encode from the slots' embedding (embed_inverse), so one vector
    encoded at several scales / levels pays for one host FFT."""
    n = ctx.n
    coeffs = emb * scale
    peak = float(np.max(np.abs(coeffs))) if coeffs.size else 0.0
    budget = ctx.level_product(level)
    if peak * 2 >= budget:
        raise EncodeRangeError(f"scaled magnitude 2^{np.log2(max(peak, 1)):.1f} exceeds the "
                               f"2^{budget.bit_length() - 1} modulus budget at level {level}")
    rounded = _round_half_away(coeffs)
    # the exact residues of the rounded coefficients (Python-integer results of
    # the reference at any magnitude) are lifted on the device from the
    # doubles themselves (fhe_real_lift): N words go up instead of L x N
    import torch

    vals = _upload_f64(ctx, rounded)
    cd = cdata_new(ctx.pool, 1, level, n, zero=False)
    _native.check(_native.lib().fhe_real_lift(ctx.chain.handle, cd.view().data_ptr(),
                                              vals.data_ptr(), n, level, 0,
                                              _native.stream_handle()), "fhe_real_lift")
    ctx.chain.transform(cd.view()[0], level, False, limbs=level, offset=0)
    cd.domains = [Domain.EVALUATION]
    return CkksPlaintext(cd, float(scale), level)


def _coeff_rows(ctx: Context, cd: CData, level: int) -> np.ndarray:
    import torch

    t = cd.view()[0].clone()
    ctx.chain.transform(t, level, True, limbs=level, offset=0)
    return t.cpu().numpy().view(np.uint64)


def ckks_decode(ctx: Context, pt: CkksPlaintext, inplace: bool = False) -> np.ndarray:
    """ckks.py:157-166: INTT, centred CRT lift to float64 and the division by
    the scale on the device (exact Python-integer float() rounding, same IEEE
    division: fhe_crt_lift), then the canonical-embedding FFT on the host
    (numpy, as the reference: bit-identical slots)."""
    from .. import _native
    from ..coremath.crt import device_lift

    # inplace: pt is a temporary (decrypt's output) and may be transformed in place
    t = pt.data.view()[0] if inplace else pt.data.view()[0].clone()
    ctx.chain.transform(t, pt.level, True, limbs=pt.level, offset=0)
    vals = device_lift(ctx, t, pt.level, _native.CRT_FLOAT, scale=pt.scale).cpu().numpy()
    if not np.isfinite(vals).all():
        raise OverflowError("int too large to convert to float")
    return embed_forward(vals, ctx.n)


# -- encrypt / decrypt ----------------------------------------------------------------

def ckks_encrypt(ctx: Context, pt: CkksPlaintext, pk: PublicKey,
                 rng: Rng | None = None) -> CkksCiphertext:
    rng = rng or Rng(fresh_seed())
    level, n = pt.level, ctx.n
    primes = ctx.q_arr(level)
    if device_sampling(ctx):  # the same Philox stream, drawn on the device
        # u, e0, e1 lifted into one (3, level, n) block and transformed by
        # one launch; e0 and e1 share one flip draw (cbd_error_pair_device)
        import torch

        uc = rng.ternary_device(n)
        e0c, e1c = rng.cbd_error_pair_device(n)
        rows = torch.empty((3, level, n), dtype=torch.int64, device="cuda")
        for k, c in enumerate((uc, e0c, e1c)):
            _native.check(_native.lib().fhe_signed_lift(ctx.chain.handle, rows[k].data_ptr(),
                                                        c.data_ptr(), n, level, 0,
                                                        _native.stream_handle()), "fhe_signed_lift")
        ctx.chain.transform(rows, 3 * level, False, limbs=level, offset=0)
        u, e0, e1 = rows[0], rows[1], rows[2]
    else:
        u = signed_eval(ctx, rng.ternary(n), primes)
        e0 = signed_eval(ctx, rng.cbd_error(n), primes)
        e1 = signed_eval(ctx, rng.cbd_error(n), primes)
    out = _new_ct(ctx, 2, level)
    v = out.view()
    pkv = pk.data.view()
    _ew(ctx, _native.EW_MUL_ADD, v[0], pkv[0, :level], u, e0, rows=level, limbs=level)
    _ew(ctx, _native.EW_ADD, v[0], v[0], pt.data.view()[0], rows=level, limbs=level)
    _ew(ctx, _native.EW_MUL_ADD, v[1], pkv[1, :level], u, e1, rows=level, limbs=level)
    return CkksCiphertext(out, pt.scale, level)


def ckks_decrypt(ctx: Context, ct: CkksCiphertext, sk: SecretKey) -> CkksPlaintext:
    import torch

    level = ct.level
    v = ct.data.view()
    s = sk.s.view()[0, :level]
    out = cdata_new(ctx.pool, 1, level, ctx.n, Domain.EVALUATION, zero=False)
    acc = out.view()[0]
    if ct.data.size_poly == 2:  # c0 + c1 s in one launch
        _ew(ctx, _native.EW_MUL_ADD, acc, v[1], s, v[0], rows=level, limbs=level)
        return CkksPlaintext(out, ct.scale, level)
    acc.copy_(v[0])
    s_pow = s
    for p in range(1, ct.data.size_poly):
        _ew(ctx, _native.EW_MUL_ADD, acc, v[p], s_pow, acc, rows=level, limbs=level)
        if p + 1 < ct.data.size_poly:
            nxt = torch.empty_like(s)
            _ew(ctx, _native.EW_MUL, nxt, s_pow, s, rows=level, limbs=level)
            s_pow = nxt
    return CkksPlaintext(out, ct.scale, level)


# -- additive ops -----------------------------------------------------------------------

def _check_pair(a, b):
    if a.level != b.level:
        raise LevelMismatch(f"levels {a.level} != {b.level}")


def _check_scales(a, b):
    if abs(a.scale - b.scale) > SCALE_RTOL * max(a.scale, b.scale):
        raise ScaleMismatch(f"scales {a.scale} and {b.scale} differ")


def ckks_add(ctx: Context, a: CkksCiphertext, b: CkksCiphertext) -> CkksCiphertext:
    _check_pair(a, b)
    _check_scales(a, b)
    pa, pb = a.data.size_poly, b.data.size_poly
    p = max(pa, pb)
    lv = a.level
    out = _new_ct(ctx, p, lv)
    common = min(pa, pb)
    # the first `common` polys start at each buffer's base: rows bound the op
    _ew(ctx, _native.EW_ADD, out._buf, a.data._buf, b.data._buf, rows=common * lv, limbs=lv)
    if p > common:
        src = a if pa > pb else b
        out.view()[common:].copy_(src.data.view()[common:])
    return CkksCiphertext(out, a.scale, lv)


def ckks_sub(ctx: Context, a: CkksCiphertext, b: CkksCiphertext) -> CkksCiphertext:
    _check_pair(a, b)
    _check_scales(a, b)
    if a.data.size_poly != b.data.size_poly:
        raise ParameterError("component-count mismatch in sub")
    out = _new_ct(ctx, a.data.size_poly, a.level)
    _ew(ctx, _native.EW_SUB, out._buf, a.data._buf, b.data._buf,
        rows=a.data.size_poly * a.level, limbs=a.level)
    return CkksCiphertext(out, a.scale, a.level)


def ckks_negate(ctx: Context, a: CkksCiphertext) -> CkksCiphertext:
    out = _new_ct(ctx, a.data.size_poly, a.level)
    _ew(ctx, _native.EW_NEG, out._buf, a.data._buf, rows=a.data.size_poly * a.level,
        limbs=a.level)
    return CkksCiphertext(out, a.scale, a.level)


def ckks_add_plain(ctx: Context, a: CkksCiphertext, pt: CkksPlaintext) -> CkksCiphertext:
    _check_pair(a, pt)
    _check_scales(a, pt)
    out = a.copy()
    v = out.data.view()
    _ew(ctx, _native.EW_ADD, v[0], v[0], pt.data.view()[0], rows=a.level, limbs=a.level)
    return out


def ckks_multiply_plain(ctx: Context, a: CkksCiphertext, pt: CkksPlaintext) -> CkksCiphertext:
    _check_pair(a, pt)
    out = _new_ct(ctx, a.data.size_poly, a.level)
    _ew(ctx, _native.EW_MUL, out._buf, a.data._buf, pt.data.view()[0],
        rows=a.data.size_poly * a.level, limbs=a.level, b_mode=_native.B_BCAST)
    return CkksCiphertext(out, a.scale * pt.scale, a.level)


class PlaintextCache:
    """Small LRU of encoded constant plaintexts (identical bits, no re-encode).

    Query circuits encode the same constants (1.0 boosts, EQ/LT coefficients,
    validity masks) hundreds of times; each host encode is an FFT, a residue
    lift, an upload and an NTT.  Plaintexts are never mutated by the ops."""

    def __init__(self, capacity: int = 512):
        from collections import OrderedDict

        self.capacity = capacity
        self._d = OrderedDict()

    def get(self, key, make):
        hit = self._d.get(key)
        if hit is not None:
            self._d.move_to_end(key)
            return hit
        val = make()
        self._d[key] = val
        if len(self._d) > self.capacity:
            self._d.popitem(last=False)
        return val


def plaintext_cache(ctx: Context) -> PlaintextCache:
    c = getattr(ctx, "_pt_cache", None)
    if c is None:
        c = PlaintextCache()
        ctx._pt_cache = c
    return c


def scalar_plaintext(ctx: Context, z: complex, scale: float, level: int) -> CkksPlaintext:
    """The two-term plaintext Re(z) + Im(z) X^(n/2) of ckks.py:290-305 (cached)."""
    return plaintext_cache(ctx).get(("scalar", complex(z), float(scale), level),
                                    lambda: _scalar_plaintext(ctx, z, scale, level))


def _scalar_plaintext(ctx: Context, z: complex, scale: float, level: int) -> CkksPlaintext:
    n = ctx.n
    coeffs = np.zeros(n)
    coeffs[0] = z.real * scale
    coeffs[n // 2] = z.imag * scale
    ints = _round_half_away(coeffs).astype(np.int64)
    rows = signed_to_residues(ints, ctx.q_arr(level))
    pt = CkksPlaintext(_poly_from_rows(ctx, rows, level), float(scale), level)
    return pt


def ckks_multiply_scalar(ctx: Context, a: CkksCiphertext, z: complex,
                         scale: float | None = None) -> CkksCiphertext:
    scale = scale or ctx.params.default_scale
    return ckks_multiply_plain(ctx, a, scalar_plaintext(ctx, complex(z), scale, a.level))


# -- multiplicative ops ------------------------------------------------------------------

def _tensor(ctx: Context, a: CkksCiphertext, b: CkksCiphertext | None) -> CData:
    lib = _native.lib()
    level = a.level
    out = _new_ct(ctx, 3, level)
    square = b is None
    _native.check(lib.fhe_tensor(ctx.chain.handle, out._buf.data_ptr(), a.data._buf.data_ptr(),
                                 None if square else b.data._buf.data_ptr(), level, 1, 0, 0, 0,
                                 1 if square else 0, _native.stream_handle()), "fhe_tensor")
    return out


def ckks_multiply(ctx: Context, a: CkksCiphertext, b: CkksCiphertext,
                  mode: str = "fused") -> CkksCiphertext:
    """Tensor product (ckks.py:308-349).  Both modes produce the same bits;
    "fused" is one fhe_tensor launch, "unfused" builds the cross term from
    separate multiply and add launches."""
    _check_pair(a, b)
    if a.data.size_poly != 2 or b.data.size_poly != 2:
        raise ParameterError("multiply requires 2-component operands")
    if mode not in ("fused", "unfused"):
        raise ParameterError(f"unknown multiply mode {mode!r}")
    if mode == "fused":
        out = _tensor(ctx, a, b)
    else:
        import torch

        lv = a.level
        out = _new_ct(ctx, 3, lv)
        x, y, o = a.data.view(), b.data.view(), out.view()
        _ew(ctx, _native.EW_MUL, o[0], x[0], y[0], rows=lv, limbs=lv)
        _ew(ctx, _native.EW_MUL, o[2], x[1], y[1], rows=lv, limbs=lv)
        t = torch.empty_like(x[0])
        _ew(ctx, _native.EW_MUL, t, x[1], y[0], rows=lv, limbs=lv)
        u = torch.empty_like(x[0])
        _ew(ctx, _native.EW_MUL, u, x[0], y[1], rows=lv, limbs=lv)
        _ew(ctx, _native.EW_ADD, o[1], u, t, rows=lv, limbs=lv)
    return CkksCiphertext(out, a.scale * b.scale, a.level)


def ckks_square(ctx: Context, a: CkksCiphertext) -> CkksCiphertext:
    if a.data.size_poly != 2:
        raise ParameterError("square requires a 2-component operand")
    return CkksCiphertext(_tensor(ctx, a, None), a.scale * a.scale, a.level)


def ckks_relinearize(ctx: Context, ct: CkksCiphertext, rlk: KSwitchKey) -> CkksCiphertext:
    if ct.data.size_poly != 3:
        raise ParameterError("relinearize expects a 3-component ciphertext")
    level = ct.level
    v = ct.data.view()
    out = _new_ct(ctx, 2, level)
    o = out.view()
    key_switch_into(ctx, level, v[2], rlk, o[0], o[1], add0=v[0], add1=v[1])
    return CkksCiphertext(out, ct.scale, level)


def ckks_multiply_relinearize(ctx: Context, a: CkksCiphertext, b: CkksCiphertext | None,
                              rlk: KSwitchKey) -> CkksCiphertext:
    """ckks_relinearize(ckks_multiply(a, b)) (or of ckks_square(a) when b is
    None) in one fused call (fhe_hmult_relin): the same words, without the
    3-component intermediate in HBM."""
    if b is None:
        b = a
    _check_pair(a, b)
    if a.data.size_poly != 2 or b.data.size_poly != 2:
        raise ParameterError("multiply requires 2-component operands")
    level = a.level
    out = _new_ct(ctx, 2, level)
    o = out.view()
    hmult_relin_into(ctx, level, a.data.view(), b.data.view(), rlk, o[0], o[1])
    return CkksCiphertext(out, a.scale * b.scale, level)


def _rescale_data(ctx: Context, data: CData, level: int, t_plain: int = 0) -> CData:
    if level < 2:
        raise LevelMismatch("rescale at level 1: level exhausted")
    lib = _native.lib()
    polys = data.size_poly
    out = cdata_new(ctx.pool, polys, level - 1, ctx.n, Domain.EVALUATION, zero=False)
    ws_bytes = lib.fhe_rescale_workspace(ctx.handle, polys, level)
    ws = ctx.workspace(ws_bytes, "rescale")
    _native.check(lib.fhe_rescale(ctx.handle, out._buf.data_ptr(), data._buf.data_ptr(), polys,
                                  level, t_plain, ws.data_ptr(), ws_bytes,
                                  _native.stream_handle()), "fhe_rescale")
    return out


def ckks_rescale(ctx: Context, ct: CkksCiphertext) -> CkksCiphertext:
    """Divide by the last chain prime with rounding and drop a level."""
    level = ct.level
    if level < 2:
        raise LevelMismatch("rescale at level 1: level exhausted")
    q_last = ctx.q_values[level - 1]
    out = _rescale_data(ctx, ct.data, level)
    return CkksCiphertext(out, ct.scale / q_last, level - 1)


def _apply_galois(ctx: Context, ct: CkksCiphertext, elt: int, gks) -> CkksCiphertext:
    if ct.data.size_poly != 2:
        raise ParameterError("rotate/conjugate expect a 2-component ciphertext")
    ksk = gks.for_elt(elt)
    level = ct.level
    perm = automorph_rows(ctx, ct.data._buf[: 2 * level * ctx.n], elt).view(2, level, ctx.n)
    out = _new_ct(ctx, 2, level)
    o = out.view()
    key_switch_into(ctx, level, perm[1], ksk, o[0], o[1], add0=perm[0], add1=None)
    return CkksCiphertext(out, ct.scale, level)


def ckks_rotate(ctx: Context, ct: CkksCiphertext, step: int, gks) -> CkksCiphertext:
    return _apply_galois(ctx, ct, ctx.galois_elt_for_step(step), gks)


def ckks_conjugate(ctx: Context, ct: CkksCiphertext, gks) -> CkksCiphertext:
    return _apply_galois(ctx, ct, ctx.conj_elt, gks)
