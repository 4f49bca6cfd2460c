"""B200-native (sm_100a) RNS-FHE hot path with the rnsfhe operator API.

Host code is Python over torch CUDA tensors; all residue arithmetic runs in
the hand-written kernels of csrc/ behind the C ABI in include/fhe_sm100.h.
"""

__version__ = "0.1.0"
