"""The Philox / bounded-integer restatement (oracle/philox.py) reproduces
numpy's Generator(Philox(SeedSequence(seed))).integers stream exactly for
the reference's three draws (sampling.py:27-63), including the state it
leaves behind (so interleaved 32- and 64-bit draws stay in step)."""
import numpy as np

from oracle.philox import PhiloxStream


def _gen(seed: int):
    return np.random.Generator(np.random.Philox(np.random.SeedSequence(seed)))


def test_stream_matches_numpy_sequence_of_reference_draws():
    seed = int.from_bytes((4).to_bytes(32, "little"), "little")
    g = _gen(seed)
    s = PhiloxStream(g.bit_generator.state)
    q = [(1 << 50) - 27, 1125899906826241, 562949953443841]
    for n in (1, 7, 64, 1000):
        for qq in q:
            want = g.integers(0, qq, size=n, dtype=np.uint64)
            assert s.integers(0, qq, n) == [int(x) for x in want]
        want = g.integers(-1, 2, size=n, dtype=np.int64)          # ternary
        assert s.integers(-1, 2, n) == [int(x) for x in want]
        want = g.integers(0, 2, size=(40, n), dtype=np.int64)     # CBD coin flips
        assert s.integers(0, 2, 40 * n) == [int(x) for x in want.reshape(-1)]
        st = g.bit_generator.state
        mine = s.state()
        assert [int(x) for x in st["state"]["counter"]] == [int(x) for x in mine["state"]["counter"]]
        assert st["buffer_pos"] == mine["buffer_pos"] and st["has_uint32"] == mine["has_uint32"]
        assert st["uinteger"] == mine["uinteger"]


def test_state_round_trip_into_numpy():
    g = _gen(12345)
    g.integers(-1, 2, size=3, dtype=np.int64)  # leaves a buffered half word
    s = PhiloxStream(g.bit_generator.state)
    a = s.integers(0, 97, 11)
    h = _gen(0)
    h.bit_generator.state = s.state()
    g.integers(0, 97, size=11, dtype=np.int64)
    assert [int(x) for x in h.integers(0, 1 << 40, size=9, dtype=np.uint64)] == \
        [int(x) for x in g.integers(0, 1 << 40, size=9, dtype=np.uint64)]
    assert len(a) == 11


def test_rejection_paths_match_numpy():
    """Ranges whose Lemire rejection rate is ~1/2 exercise the resampling
    loops of both bounded paths (sampling draws never hit them in practice)."""
    g = _gen(99)
    s = PhiloxStream(g.bit_generator.state)
    for lo, hi, n in ((0, (1 << 63) + 1, 500), (0, (1 << 31) + 1, 500), (-5, 3, 77),
                      (0, 1 << 62, 33), (0, (1 << 32) - 1, 50)):
        want = g.integers(lo, hi, size=n, dtype=np.uint64 if lo >= 0 else np.int64)
        assert s.integers(lo, hi, n) == [int(x) for x in want], (lo, hi)
