"""ctypes binding of libfhe_sm100.so (include/fhe_sm100.h).

The product path has no CPU fallback: importing works anywhere (so the CPU
test-suite can check the exported symbols), but every compute entry point
raises NativeUnavailable when the library or a CUDA device is missing.
"""

from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FHE_SM100_LIB") or os.path.join(_HERE, "lib", "libfhe_sm100.so")
HEADER_PATH = os.path.join(os.path.dirname(_HERE), "include", "fhe_sm100.h")

# op codes / operand modes (mirror include/fhe_sm100.h)
CRT_FLOAT, CRT_MOD_T, CRT_BFV = range(3)
EW_ADD, EW_SUB, EW_NEG, EW_MUL, EW_NEG_MUL, EW_MUL_ADD, EW_MUL_SUB, EW_REDUCE = range(8)
B_FULL, B_BCAST, B_CONST = range(3)
# NTT kernel paths (fhe_ntt_path_count)
NTT_PATHS = {"rows": 0, "split": 1, "fused_tma": 2, "fused_cp": 3, "int": 4, "cluster": 5,
             "mm": 6}

_u64p = ctypes.c_void_p
_vp = ctypes.c_void_p
_i64 = ctypes.c_int64
_int = ctypes.c_int
_sz = ctypes.c_size_t

# name -> (restype, argtypes)
SIGNATURES = {
    "fhe_last_error": (ctypes.c_char_p, []),
    "fhe_launch_count": (ctypes.c_uint64, []),
    "fhe_device_sm_count": (_int, []),
    "fhe_ntt_path_count": (ctypes.c_uint64, [_int]),
    "fhe_chain_create": (_int, [_vp, _int, _int, ctypes.POINTER(_vp)]),
    "fhe_chain_destroy": (_int, [_vp]),
    "fhe_chain_tables": (_int, [_vp, _int, _vp, _vp, _vp, _vp]),
    "fhe_ntt_fwd": (_int, [_vp, _u64p, _i64, _vp, _int, _int, _vp]),
    "fhe_ntt_inv": (_int, [_vp, _u64p, _i64, _vp, _int, _int, _vp]),
    "fhe_ntt_mm": (_int, [_vp, _u64p, _u64p, _i64, _vp, _int, _int, _int, _vp]),
    "fhe_ewise": (_int, [_vp, _int, _u64p, _u64p, _u64p, _u64p, _i64, _vp, _int, _int, _int,
                         _vp]),
    "fhe_tensor": (_int, [_vp, _u64p, _u64p, _u64p, _int, _i64, _i64, _i64, _i64, _int, _vp]),
    "fhe_automorph": (_int, [_u64p, _u64p, _i64, _int, ctypes.c_uint64, _vp]),
    "fhe_context_create": (_int, [_vp, _int, _vp, _int, _int, _int, ctypes.POINTER(_vp)]),
    "fhe_context_destroy": (_int, [_vp]),
    "fhe_context_prepare_plain": (_int, [_vp, ctypes.c_uint64]),
    "fhe_philox_workspace": (ctypes.c_size_t, [ctypes.c_int64, ctypes.c_uint64]),
    "fhe_philox_integers": (_int, [_vp, ctypes.c_int64, ctypes.c_uint64, ctypes.c_int64, _vp, _vp,
                                   _sz, _vp]),
    "fhe_cbd_combine": (_int, [_vp, _vp, _int, ctypes.c_int64, _vp]),
    "fhe_real_lift": (_int, [_vp, _vp, _vp, ctypes.c_int64, _int, _int, _vp]),
    "fhe_signed_lift": (_int, [_vp, _vp, _vp, ctypes.c_int64, _int, _int, _vp]),
    "fhe_crc32_workspace": (ctypes.c_size_t, [ctypes.c_int64]),
    "fhe_crc32": (_int, [_vp, ctypes.c_int64, _vp, _vp, _sz, _vp]),
    "fhe_crt_lift": (_int, [_vp, _int, _vp, _vp, _int, ctypes.c_double, ctypes.c_uint64,
                            ctypes.c_uint64, _vp]),
    "fhe_context_chain": (_vp, [_vp]),
    "fhe_rescale_workspace": (_sz, [_vp, _int, _int]),
    "fhe_rescale": (_int, [_vp, _u64p, _u64p, _int, _int, ctypes.c_uint64, _vp, _sz, _vp]),
    "fhe_keyswitch_workspace": (_sz, [_vp, _int, _int]),
    "fhe_behz_lift": (_int, [_vp, _u64p, _u64p, _int, _int, _int, _u64p, _vp]),
    "fhe_behz_floor": (_int, [_vp, _u64p, _u64p, _int, _int, _int, _u64p, _vp]),
    "fhe_keyswitch": (_int, [_vp, _int, _u64p, _i64, _u64p, _u64p, _u64p, _i64, _u64p, _u64p,
                             _i64, _int, _vp, _sz, _vp]),
    "fhe_hmult_relin_workspace": (_sz, [_vp, _int, _int]),
    "fhe_hmult_relin": (_int, [_vp, _int, _u64p, _u64p, _i64, _u64p, _u64p, _u64p, _i64, _int,
                               _vp, _sz, _vp]),
}


class NativeUnavailable(RuntimeError):
    """The sm_100a library or a CUDA device is not available."""


class NativeError(RuntimeError):
    """A native entry point returned an error code."""


_lib = None


def load_library(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load the shared library and declare every prototype (no GPU needed)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise NativeUnavailable(
            f"{path} not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = ctypes.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


_device_ok = False


def lib() -> ctypes.CDLL:
    """Library handle for compute calls: requires a CUDA device (probed once;
    the answer cannot change inside a process)."""
    global _device_ok
    if not _device_ok:
        import torch

        if not torch.cuda.is_available():
            raise NativeUnavailable("no CUDA device: the B200 path has no CPU fallback")
        _device_ok = True
    return _lib if _lib is not None else load_library()


def ntt_path_counts() -> dict:
    """Transform launches per NTT kernel path so far (fhe_ntt_path_count)."""
    lb = load_library()
    return {k: int(lb.fhe_ntt_path_count(v)) for k, v in NTT_PATHS.items()}


def check(rc: int, what: str):
    if rc != 0:
        msg = load_library().fhe_last_error()
        raise NativeError(f"{what} failed ({rc}): {msg.decode() if msg else ''}")


def stream_handle(stream=None) -> int:
    """cudaStream_t of `stream`, else of torch's current stream on the current
    device (read through torch's raw accessor: no Stream object per call)."""
    import torch

    if stream is not None:
        return stream.cuda_stream
    return torch._C._cuda_getCurrentRawStream(torch._C._cuda_getDevice())


def ptr(t) -> int:
    """Device address of a torch tensor (or an int passthrough)."""
    if t is None:
        return None
    if isinstance(t, int):
        return t
    return t.data_ptr()
