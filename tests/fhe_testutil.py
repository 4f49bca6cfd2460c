"""Shared helpers for the test-suite (import as fhe_testutil)."""

import hashlib
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def digest(a) -> str:
    """SHA-256 of an array's little-endian uint64 words (tests/golden format)."""
    if hasattr(a, "detach"):
        a = a.detach().cpu().numpy()
    a = np.ascontiguousarray(np.asarray(a).view(np.uint64) if np.asarray(a).dtype == np.int64
                             else np.asarray(a, dtype=np.uint64))
    return hashlib.sha256(a.astype("<u8").tobytes()).hexdigest()


def to_u64(t) -> np.ndarray:
    if hasattr(t, "detach"):
        return t.detach().cpu().numpy().view(np.uint64)
    return np.asarray(t, dtype=np.uint64)


def seeded_rng(seed: int = 1234):
    from paper_2503_22227_b200.coremath.sampling import Rng

    return Rng(int(seed).to_bytes(32, "little"))
