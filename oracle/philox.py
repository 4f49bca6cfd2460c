"""Test infrastructure only (not product code): a pure-Python restatement of
the third-party sampler the reference uses for keys and noise -- numpy
2.3.5's Generator(Philox(SeedSequence(seed))) -- pinned against numpy itself
by tests/test_philox_oracle.py.

The reference draws through rnsfhe/coremath/sampling.py:27-63:
  uniform_residues: Generator.integers(0, q, n, uint64)   (64-bit Lemire)
  ternary:          Generator.integers(-1, 2, n, int64)   (32-bit Lemire)
  cbd_error:        Generator.integers(0, 2, (40, n), int64)
numpy's algorithms restated here (numpy/random/src/philox/philox.h,
numpy/random/src/distributions/distributions.c random_bounded_uint64_fill,
bounded_lemire_uint64, buffered_bounded_lemire_uint32):
  * Philox4x64-10 (Random123): 10 rounds of the two 64x64->128 products with
    M0 = 0xD2E7470EE14C6C93, M1 = 0xCA5A826395121157 and the key bumped by
    W0 = 0x9E3779B97F4A7C15, W1 = 0xBB67AE8584CAA73B between rounds;
  * next_uint64: serve buffer[buffer_pos++]; when empty, increment the
    256-bit counter FIRST, then refill all 4 words (buffer_pos = 1);
  * next_uint32: the low half of a 64-bit draw, its high half kept in
    (has_uint32, uinteger) for the next 32-bit draw;
  * Lemire: m = draw * (rng + 1); reject while low part < (MAX - rng) % (rng + 1)
    (only tested when low part < rng + 1); value = off + high part.
The device sampler (csrc/philox.cu) implements the same stream.
"""

from __future__ import annotations

M0, M1 = 0xD2E7470EE14C6C93, 0xCA5A826395121157
W0, W1 = 0x9E3779B97F4A7C15, 0xBB67AE8584CAA73B
MASK64 = (1 << 64) - 1


def philox4x64(ctr, key, rounds=10):
    c = list(ctr)
    k0, k1 = key
    for r in range(rounds):
        if r:
            k0 = (k0 + W0) & MASK64
            k1 = (k1 + W1) & MASK64
        p0 = M0 * c[0]
        p1 = M1 * c[2]
        hi0, lo0 = p0 >> 64, p0 & MASK64
        hi1, lo1 = p1 >> 64, p1 & MASK64
        c = [hi1 ^ c[1] ^ k0, lo1, hi0 ^ c[3] ^ k1, lo0]
    return c


class PhiloxStream:
    """numpy's Philox bit generator state machine (state dict round trip)."""

    def __init__(self, state: dict):
        st = state["state"]
        self.ctr = [int(x) for x in st["counter"]]
        self.key = [int(x) for x in st["key"]]
        self.buffer = [int(x) for x in state["buffer"]]
        self.buffer_pos = int(state["buffer_pos"])
        self.has_uint32 = int(state["has_uint32"])
        self.uinteger = int(state["uinteger"])

    def state(self) -> dict:
        import numpy as np

        return {"bit_generator": "Philox",
                "state": {"counter": np.array(self.ctr, dtype=np.uint64),
                          "key": np.array(self.key, dtype=np.uint64)},
                "buffer": np.array(self.buffer, dtype=np.uint64),
                "buffer_pos": self.buffer_pos, "has_uint32": self.has_uint32,
                "uinteger": self.uinteger}

    def next64(self) -> int:
        if self.buffer_pos < 4:
            v = self.buffer[self.buffer_pos]
            self.buffer_pos += 1
            return v
        for i in range(4):  # 256-bit increment
            self.ctr[i] = (self.ctr[i] + 1) & MASK64
            if self.ctr[i]:
                break
        self.buffer = philox4x64(self.ctr, self.key)
        self.buffer_pos = 1
        return self.buffer[0]

    def next32(self) -> int:
        if self.has_uint32:
            self.has_uint32 = 0
            return self.uinteger
        v = self.next64()
        self.has_uint32 = 1
        self.uinteger = v >> 32
        return v & 0xFFFFFFFF

    # Generator.integers(low, high, size) for size elements (endpoint=False)
    def integers(self, low: int, high: int, size: int) -> list[int]:
        rng = high - low - 1
        out = []
        if rng == 0:
            return [low] * size
        if rng <= 0xFFFFFFFF:
            excl = rng + 1
            thr = (0xFFFFFFFF - rng) % excl
            for _ in range(size):
                if rng == 0xFFFFFFFF:
                    out.append(low + self.next32())
                    continue
                m = self.next32() * excl
                left = m & 0xFFFFFFFF
                if left < excl:
                    while left < thr:
                        m = self.next32() * excl
                        left = m & 0xFFFFFFFF
                out.append(low + (m >> 32))
            return out
        excl = rng + 1
        thr = (MASK64 - rng) % excl
        for _ in range(size):
            m = self.next64() * excl
            left = m & MASK64
            if left < excl:
                while left < thr:
                    m = self.next64() * excl
                    left = m & MASK64
            out.append(low + (m >> 64))
        return out
