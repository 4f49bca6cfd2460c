"""Drop-in for the reference's kernel seam ``rnsfhe.coremath._kernels``
(coremath/_kernels.py:86-173), the module the reference imports behind
try/except at its five call sites (ntt.py:24-27, rnspoly.py:21-24,
keys.py:22-25, ckks.py:33-36, behz.py:22-25).

Same function names, argument order and semantics: host numpy arrays,
(rows, n) uint64 C-contiguous, per-chain tables indexed by ``mod_idx``,
results written IN PLACE (``a`` for the transforms, ``out`` for the
products), no return value.  The arithmetic runs on the B200 through
libfhe_sm100 (fhe_ntt_fwd / fhe_ntt_inv / fhe_ewise): each call uploads its
operands, runs the batched kernel and copies the result back into the
caller's array.  The reference's numba kernels have no error channel; this
module raises (ValueError / NativeUnavailable) instead of computing anything
on the host -- there is no CPU fallback.

The reference passes its own tables (psi, Shoup companions, Montgomery
qinv / r2).  The device chain is built from ``q`` (and the degree) and owns
equivalent tables; on first use of a chain the passed psi rows are checked
against the device's (psi = smallest primitive 2N-th root, ntt.py:72), so a
caller with different tables fails loudly instead of getting other words.
Montgomery constants are not needed by the exact device products (any exact
product mod q gives the same canonical word).

A maintainer enables it by replacing the body of rnsfhe/coremath/_kernels.py
with ``from paper_2503_22227_b200.coremath._kernels import *``.
"""

from __future__ import annotations

import numpy as np

from .. import _native
from .ntt import DeviceChain

__all__ = ["ntt_batch", "intt_batch", "mul_batch", "neg_mul_batch", "mul_add_batch"]

_chains: dict = {}      # (q tuple, n) -> DeviceChain
_checked: set = set()   # (q tuple, n, direction) whose psi tables were verified


def _chain(q, n: int) -> DeviceChain:
    key = (tuple(int(v) for v in np.asarray(q, dtype=np.uint64)), int(n))
    ch = _chains.get(key)
    if ch is None:
        if n < 2 or n & (n - 1):
            raise ValueError(f"row length {n} is not a power of two")
        ch = DeviceChain(list(key[0]), n.bit_length() - 1)
        _chains[key] = ch
    return ch


def _check_tables(ch: DeviceChain, tables, inverse: bool):
    key = (tuple(ch.primes), ch.n, inverse)
    if key in _checked:
        return
    tables = np.asarray(tables, dtype=np.uint64)
    if tables.shape != (len(ch.primes), ch.n):
        raise ValueError(f"twiddle table shape {tables.shape} != ({len(ch.primes)}, {ch.n})")
    for j in range(len(ch.primes)):
        _, fw, iv, _ = ch.tables(j)
        if not np.array_equal(tables[j], iv if inverse else fw):
            raise ValueError(f"twiddle table of chain position {j} differs from the device "
                             "chain's (psi must be the smallest primitive 2N-th root)")
    _checked.add(key)


def _rows(a: np.ndarray, what: str) -> np.ndarray:
    if not isinstance(a, np.ndarray) or a.ndim != 2 or a.dtype != np.uint64:
        raise ValueError(f"{what} must be a (rows, n) uint64 array")
    if not a.flags.c_contiguous:
        raise ValueError(f"{what} must be C-contiguous")
    return a


def _dev(a: np.ndarray):
    import torch

    return torch.from_numpy(a.view(np.int64)).cuda()


def _store(dst: np.ndarray, dev) -> None:
    import torch

    if not dst.flags.writeable:
        raise ValueError("output array is read-only")
    torch.from_numpy(dst.view(np.int64)).copy_(dev.cpu())


def _transform(a, tables, q, mod_idx, inverse: bool):
    _native.lib()  # fails loudly without a device / the library
    a = _rows(a, "a")
    rows, n = a.shape
    ch = _chain(q, n)
    _check_tables(ch, tables, inverse)
    if rows == 0:
        return
    d = _dev(a)
    ch.transform(d, rows, inverse, np.asarray(mod_idx, dtype=np.int64))
    _store(a, d)


def ntt_batch(a, psi, psi_sh, q, mod_idx):
    """Forward negacyclic NTT of every row of a, in place (_kernels.py:88-92)."""
    _transform(a, psi, q, mod_idx, inverse=False)


def intt_batch(a, ipsi, ipsi_sh, n_inv, n_inv_sh, q, mod_idx):
    """Inverse NTT (with n^-1) of every row of a, in place (_kernels.py:95-99)."""
    _transform(a, ipsi, q, mod_idx, inverse=True)


def _ewise(op, a, b, c, out, q, mod_idx):
    lib = _native.lib()
    a = _rows(a, "a")
    b = _rows(b, "b")
    out = _rows(out, "out")
    if c is not None:
        c = _rows(c, "c")
    rows, n = a.shape
    for name, x in (("b", b), ("out", out), ("c", c)):
        if x is not None and x.shape != a.shape:
            raise ValueError(f"{name} shape {x.shape} != a shape {a.shape}")
    if rows == 0:
        return
    ch = _chain(q, n)
    idx, limbs, offset = ch._rowmap(rows, np.asarray(mod_idx, dtype=np.int64))
    da, db = _dev(a), _dev(b)
    dc = _dev(c) if c is not None else None
    dout = da.new_empty(da.shape)
    _native.check(lib.fhe_ewise(ch.handle, op, dout.data_ptr(), da.data_ptr(), db.data_ptr(),
                                dc.data_ptr() if dc is not None else None, rows, idx,
                                limbs, offset, _native.B_FULL, _native.stream_handle()),
                  "fhe_ewise")
    _store(out, dout)


def mul_batch(a, b, out, q, qinv, r2, mod_idx):
    """out = a * b mod q_(mod_idx[r]) (_kernels.py:141-150)."""
    _ewise(_native.EW_MUL, a, b, None, out, q, mod_idx)


def neg_mul_batch(a, b, out, q, qinv, r2, mod_idx):
    """out = -(a * b) mod q (_kernels.py:153-163)."""
    _ewise(_native.EW_NEG_MUL, a, b, None, out, q, mod_idx)


def mul_add_batch(a, b, c, out, q, qinv, r2, mod_idx):
    """out = a * b + c mod q (_kernels.py:166-176)."""
    _ewise(_native.EW_MUL_ADD, a, b, c, out, q, mod_idx)
