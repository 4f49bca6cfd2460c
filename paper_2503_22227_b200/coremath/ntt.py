"""Batched negacyclic NTT over an RNS chain on the B200.

Drop-in for the reference's ``NttChain`` (coremath/ntt.py:240-351): the same
(rows, n) residue-row interface with a per-row ``mod_idx``, the same
bit-reversed output order and the same canonical residues.  The work runs in
the sm_100a kernels of csrc/ntt.cu; numpy inputs are uploaded, transformed on
the device and returned as numpy (convenience for tests and host code), torch
CUDA tensors are transformed without leaving HBM.
"""

from __future__ import annotations

import ctypes
from enum import Enum

import numpy as np

from .. import _native
from .modmath import Modulus, ParameterError

MATRIX_DEGREE_LIMIT = 1024


class ShapeError(ValueError):
    pass


class ConfigurationError(RuntimeError):
    """The matrix variant was requested without materialize_matrix()
    (reference ntt.py:34-35)."""


class NttVariant(str, Enum):
    AUTO = "auto"
    FORCE_BM = "force_bm"
    FORCE_MM = "force_mm"


def bit_reverse(x: int, bits: int) -> int:
    r = 0
    for _ in range(bits):
        r = (r << 1) | (x & 1)
        x >>= 1
    return r


def exponent_map(n: int) -> np.ndarray:
    """exp[j]: NTT slot j holds the evaluation at psi^exp[j] (ntt.py:128-137)."""
    bits = n.bit_length() - 1
    j = np.arange(n, dtype=np.int64)
    rev = np.zeros(n, dtype=np.int64)
    for b in range(bits):
        rev |= ((j >> b) & 1) << (bits - 1 - b)
    return 2 * rev + 1


class DeviceChain:
    """Owner of one native FheChain (tables resident in HBM)."""

    def __init__(self, primes, log_n: int, handle=None, owner=None):
        self.primes = [int(p.value if isinstance(p, Modulus) else p) for p in primes]
        self.log_n = log_n
        self.n = 1 << log_n
        self._owner = owner
        if handle is None:
            lib = _native.lib()
            arr = (ctypes.c_uint64 * len(self.primes))(*self.primes)
            h = ctypes.c_void_p()
            _native.check(lib.fhe_chain_create(arr, len(self.primes), log_n, ctypes.byref(h)),
                          "fhe_chain_create")
            self.handle = h.value
            self._owns = True
        else:
            self.handle = handle
            self._owns = False
        self._idx_cache: dict = {}

    def __del__(self):
        try:
            if self._owns and self.handle:
                _native.load_library().fhe_chain_destroy(self.handle)
        except Exception:  # pragma: no cover - interpreter teardown
            pass

    def tables(self, idx: int):
        """(psi, psi_br, ipsi_br, n_inv) host copies of one prime's tables."""
        lib = _native.lib()
        n = self.n
        psi = ctypes.c_uint64()
        ninv = ctypes.c_uint64()
        fw = np.empty(n, dtype=np.uint64)
        iv = np.empty(n, dtype=np.uint64)
        _native.check(lib.fhe_chain_tables(self.handle, idx, ctypes.byref(psi),
                                           fw.ctypes.data, iv.ctypes.data, ctypes.byref(ninv)),
                      "fhe_chain_tables")
        return int(psi.value), fw, iv, int(ninv.value)

    # -- device-side row maps ---------------------------------------------------
    def mod_idx_tensor(self, mod_idx):
        import torch

        key = mod_idx.tobytes() if isinstance(mod_idx, np.ndarray) else tuple(mod_idx)
        t = self._idx_cache.get(key)
        if t is None:
            t = torch.as_tensor(np.asarray(mod_idx, dtype=np.int32), device="cuda")
            self._idx_cache[key] = t
        return t

    def _rowmap(self, rows: int, mod_idx):
        """(device idx pointer or None, limbs, offset) for a row map."""
        if mod_idx is None:
            return None, len(self.primes), 0
        mi = np.asarray(mod_idx, dtype=np.int64)
        if mi.shape[0] != rows:
            raise ShapeError("mod_idx length does not match row count")
        if mi.size and (mi.min() < 0 or mi.max() >= len(self.primes)):
            raise ShapeError("mod_idx outside the chain")
        # detect the layout-order pattern (r % limbs) + offset
        if rows:
            off = int(mi[0])
            limbs = 1
            while limbs < rows and mi[limbs] == off + limbs:
                limbs += 1
            if np.array_equal(mi, (np.arange(rows) % limbs) + off):
                return None, limbs, off
        return self.mod_idx_tensor(mi.astype(np.int32)).data_ptr(), rows, 0

    def transform(self, data, rows: int, inverse: bool, mod_idx=None, limbs=None, offset=0,
                  stream=None):
        """In-place transform of ``rows`` contiguous device rows (torch tensor or
        address)."""
        lib = _native.lib()
        if limbs is None:
            idx, limbs, offset = self._rowmap(rows, mod_idx)
        else:
            idx = None
        fn = lib.fhe_ntt_inv if inverse else lib.fhe_ntt_fwd
        _native.check(fn(self.handle, _native.ptr(data), rows, idx, limbs, offset,
                         _native.stream_handle(stream)), "fhe_ntt")

    def transform_mm(self, out, data, rows: int, inverse: bool, mod_idx=None, stream=None):
        """Matrix-product variant (fhe_ntt_mm) of ``rows`` device rows into
        ``out`` (must not alias ``data``)."""
        lib = _native.lib()
        idx, limbs, offset = self._rowmap(rows, mod_idx)
        _native.check(lib.fhe_ntt_mm(self.handle, _native.ptr(out), _native.ptr(data), rows, idx,
                                     limbs, offset, int(bool(inverse)),
                                     _native.stream_handle(stream)), "fhe_ntt_mm")


class NttTables:
    """Per-(degree, modulus) tables, read back from the device chain
    (reference NttTables, ntt.py:52-137)."""

    def __init__(self, degree: int, modulus):
        if degree < 2 or degree & (degree - 1):
            raise ParameterError(f"degree {degree} is not a power of two")
        m = modulus if isinstance(modulus, Modulus) else Modulus(int(modulus))
        if (m.value - 1) % (2 * degree):
            raise ParameterError(f"{m.value} is not NTT friendly for degree {degree}")
        self.degree = degree
        self.modulus = m
        self._chain = DeviceChain([m.value], degree.bit_length() - 1)
        self.psi, self.psi_powers, self.inv_psi_powers, self.n_inv = self._chain.tables(0)
        self.dft_matrix = None
        self.inv_dft_matrix = None

    def exponent_map(self) -> np.ndarray:
        return exponent_map(self.degree)

    def materialize_matrix(self):
        """Enable the matrix variant (reference ntt.py:101-124).  The device
        kernel reads every entry psi^(exp_j * i) from the psi table, so the
        n x n matrices are not stored: the attributes only record that the
        variant was set up (ntt_mm raises ConfigurationError before)."""
        if self.degree > 1 << 13:
            raise ParameterError("matrix NTT variant supports degree <= 2^13")
        self.dft_matrix = "device"
        self.inv_dft_matrix = "device"


class NttChain:
    """Stacked transforms over a modulus chain (reference ntt.py:240-351)."""

    def __init__(self, moduli, degree: int | None = None, variant=NttVariant.AUTO,
                 device_chain: DeviceChain | None = None):
        if device_chain is None:
            if isinstance(moduli, (list, tuple)) and moduli and isinstance(moduli[0], NttTables):
                degree = moduli[0].degree
                moduli = [t.modulus for t in moduli]
            if not moduli or degree is None:
                raise ParameterError("empty table chain")
            device_chain = DeviceChain(moduli, degree.bit_length() - 1)
        self.dev = device_chain
        self.degree = device_chain.n
        self.variant = NttVariant(variant)
        self.q = np.array(device_chain.primes, dtype=np.uint64)

    def _run(self, a, mod_idx, inverse: bool):
        import torch

        if a.ndim != 2 or a.shape[1] != self.degree:
            raise ShapeError(f"expected (rows, {self.degree}), got {tuple(a.shape)}")
        rows = a.shape[0]
        if mod_idx is None:
            mod_idx = np.arange(rows) % len(self.dev.primes)
        mm = self.variant is NttVariant.FORCE_MM
        if isinstance(a, torch.Tensor):
            src = a.contiguous()
        else:
            host = np.ascontiguousarray(a, dtype=np.uint64)
            src = torch.from_numpy(host.view(np.int64)).cuda()
        if mm:
            # forced matrix variant (reference NttChain._per_row -> ntt_dispatch,
            # ntt.py:266-275): same words as the butterflies
            out = torch.empty_like(src)
            self.dev.transform_mm(out, src, rows, inverse, mod_idx)
        else:
            out = src.clone() if isinstance(a, torch.Tensor) else src
            self.dev.transform(out, rows, inverse, mod_idx)
        return out if isinstance(a, torch.Tensor) else out.cpu().numpy().view(np.uint64)

    def forward(self, a, mod_idx=None):
        return self._run(a, mod_idx, inverse=False)

    def inverse(self, a, mod_idx=None):
        return self._run(a, mod_idx, inverse=True)


# -- single-row transforms and the variant dispatch (reference ntt.py:145-233,
#    354-364); every variant runs on the device and returns canonical words.


def _single(vec, tables: NttTables, inverse: bool, mm: bool):
    import torch

    v = np.asarray(vec)
    if v.shape != (tables.degree,):
        raise ShapeError(f"expected length {tables.degree}, got {v.shape}")
    if mm and tables.dft_matrix is None:
        raise ConfigurationError("dft matrix not materialized; call materialize_matrix()")
    src = torch.from_numpy(np.ascontiguousarray(v, dtype=np.uint64).view(np.int64)).cuda()
    src = src.reshape(1, -1)
    if mm:
        out = torch.empty_like(src)
        tables._chain.transform_mm(out, src, 1, inverse)
    else:
        out = src
        tables._chain.transform(out, 1, inverse)
    return out.cpu().numpy().view(np.uint64).reshape(-1)


def ntt_bm(coeffs, tables: NttTables) -> np.ndarray:
    """Forward negacyclic NTT, butterflies (reference ntt.py:145-169)."""
    return _single(coeffs, tables, False, False)


def intt_bm(evals, tables: NttTables) -> np.ndarray:
    """Inverse of ntt_bm (reference ntt.py:172-198)."""
    return _single(evals, tables, True, False)


def ntt_mm(coeffs, tables: NttTables) -> np.ndarray:
    """Forward NTT as an n x n matrix-vector product (reference ntt.py:220-225)."""
    return _single(coeffs, tables, False, True)


def intt_mm(evals, tables: NttTables) -> np.ndarray:
    """Inverse matrix variant (reference ntt.py:228-233)."""
    return _single(evals, tables, True, True)


def ntt_dispatch(coeffs, tables: NttTables, policy=NttVariant.AUTO,
                 inverse: bool = False) -> np.ndarray:
    """Matrix product below degree 1024, butterflies above (reference
    ntt.py:354-364)."""
    policy = NttVariant(policy)
    if policy is NttVariant.FORCE_MM or (policy is NttVariant.AUTO
                                         and tables.degree < MATRIX_DEGREE_LIMIT):
        if tables.dft_matrix is None:
            tables.materialize_matrix()
        return intt_mm(coeffs, tables) if inverse else ntt_mm(coeffs, tables)
    return intt_bm(coeffs, tables) if inverse else ntt_bm(coeffs, tables)
