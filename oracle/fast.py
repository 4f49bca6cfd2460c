"""ctypes front-end of oracle/c/fhe_oracle.c - TEST INFRASTRUCTURE ONLY.

Same call signatures as oracle/rns_oracle.py for the functions both provide;
used for full-size parity checks and the CPU baseline.  Built by
`make -C oracle` (run from __graft_entry__.build())."""

from __future__ import annotations

import ctypes
import os

import numpy as np

_LIB = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_build", "libfhe_oracle.so")
_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB):
            raise RuntimeError(f"{_LIB} missing: run `make -C oracle`")
        _lib = ctypes.CDLL(_LIB)
        vp, i, lg = ctypes.c_void_p, ctypes.c_int, ctypes.c_long
        _lib.orc_ntt.argtypes = [vp, lg, i, vp, i, vp, i]
        _lib.orc_tensor.argtypes = [vp, vp, vp, i, i, vp]
        _lib.orc_add.argtypes = [vp, vp, vp, i, i, i, vp]
        _lib.orc_keyswitch.argtypes = [vp, i, i, vp, vp, i, vp, i, i, vp, vp]
        _lib.orc_keyswitch.restype = i
        _lib.orc_rescale.argtypes = [vp, vp, i, i, i, vp]
        _lib.orc_threads.restype = i
    return _lib


def threads() -> int:
    return lib().orc_threads()


def _u64(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.uint64))


def _primes(p):
    return _u64([int(x) for x in p])


def _log(n):
    return int(n).bit_length() - 1


def ntt_forward(a, primes, mod_idx=None, inverse=False):
    out = _u64(a).copy()
    pr = _primes(primes)
    mi = None if mod_idx is None else np.ascontiguousarray(mod_idx, dtype=np.int32)
    lib().orc_ntt(out.ctypes.data, out.shape[0], _log(out.shape[1]), pr.ctypes.data, len(pr),
                  None if mi is None else mi.ctypes.data, 1 if inverse else 0)
    return out


def ntt_inverse(a, primes, mod_idx=None):
    return ntt_forward(a, primes, mod_idx, inverse=True)


def tensor(x, y, primes):
    x, y = _u64(x), _u64(y)
    _, L, n = x.shape
    out = np.empty((3, L, n), dtype=np.uint64)
    pr = _primes(primes)
    lib().orc_tensor(out.ctypes.data, x.ctypes.data, y.ctypes.data, L, _log(n), pr.ctypes.data)
    return out[0], out[1], out[2]


def add(a, b, primes):
    a, b = _u64(a), _u64(b)
    out = np.empty_like(a)
    L, n = a.shape[-2], a.shape[-1]
    polys = a.size // (L * n)
    pr = _primes(primes)
    lib().orc_add(out.ctypes.data, a.ctypes.data, b.ctypes.data, polys, L, _log(n),
                  pr.ctypes.data)
    return out


def key_switch(d, keys, primes, alpha=1, special=()):
    d, keys = _u64(d), _u64(keys)
    level, n = d.shape
    Q, P = _primes(primes), _primes(list(special) or [0])
    b = np.empty((level, n), dtype=np.uint64)
    a = np.empty((level, n), dtype=np.uint64)
    rc = lib().orc_keyswitch(d.ctypes.data, level, _log(n), keys.ctypes.data, Q.ctypes.data,
                             len(Q), P.ctypes.data, len(special), alpha, b.ctypes.data,
                             a.ctypes.data)
    if rc:
        raise ValueError("oracle key switch: alpha/K too large")
    return b, a


def rescale(ct, primes):
    ct = _u64(ct)
    polys, L, n = ct.shape
    out = np.empty((polys, L - 1, n), dtype=np.uint64)
    pr = _primes(primes)
    lib().orc_rescale(out.ctypes.data, ct.ctypes.data, polys, L, _log(n), pr.ctypes.data)
    return out
