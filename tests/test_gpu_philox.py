"""Device sampler (csrc/philox.cu) against numpy's own Generator stream and
against the host path: the same seeds give the same words, in the
reference's call order (sampling.py:27-63), with host and device draws
interleaved, and across Lemire rejections (heavy-rejection ranges)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _pair(seed):
    from paper_2503_22227_b200.coremath.sampling import Rng

    return (Rng(int(seed).to_bytes(32, "little")),
            np.random.Generator(np.random.Philox(np.random.SeedSequence(seed))))


def test_reference_draw_sequence_on_device():
    r, g = _pair(4)
    q = [(1 << 50) - 27, 1125899906826241, 562949953443841, (1 << 60) + 33]
    for n in (1, 5, 4096, 65536 + 3):
        got = r.uniform_residues_device(q, n).cpu().numpy().view(np.uint64)
        want = np.stack([g.integers(0, qq, size=n, dtype=np.uint64) for qq in q])
        assert np.array_equal(got, want), n
        assert np.array_equal(r.ternary_device(n).cpu().numpy(),
                              g.integers(-1, 2, size=n, dtype=np.int64))
        flips = g.integers(0, 2, size=(40, n), dtype=np.int64)
        assert np.array_equal(r.cbd_error_device(n).cpu().numpy(),
                              flips[:20].sum(axis=0) - flips[20:].sum(axis=0))


def test_host_and_device_draws_interleave():
    r, g = _pair(77)
    a = r.ternary(3)                                    # host, leaves a buffered half word
    b = r.integers_device(0, 1 << 45, 10).cpu().numpy()  # device
    c = r.cbd_error(7)                                  # host again (state comes back)
    d = r.ternary_device(9).cpu().numpy()
    e = r.uniform_bytes(16)
    assert np.array_equal(a, g.integers(-1, 2, size=3, dtype=np.int64))
    assert np.array_equal(b, g.integers(0, 1 << 45, size=10, dtype=np.int64))
    flips = g.integers(0, 2, size=(40, 7), dtype=np.int64)
    assert np.array_equal(c, flips[:20].sum(axis=0) - flips[20:].sum(axis=0))
    assert np.array_equal(d, g.integers(-1, 2, size=9, dtype=np.int64))
    assert e == g.bytes(16)


def test_rejection_heavy_ranges():
    r, g = _pair(5)
    for lo, hi, n in ((0, (1 << 31) + 1, 3000), (0, (1 << 62) + 1, 100)):
        got = r.integers_device(lo, hi, n).cpu().numpy().view(np.uint64)
        assert np.array_equal(got, g.integers(lo, hi, size=n, dtype=np.uint64))


def test_cbd_pair_draw_equals_two_host_draws():
    """cbd_error_pair_device (one flip draw for e0 and e1, ckks_encrypt) gives
    the words of two consecutive host cbd_error draws and leaves the stream
    where they leave it."""
    from paper_2503_22227_b200.coremath.sampling import Rng

    for seed, n in ((11, 4096), (12, 1 << 16), (13, 17)):
        a = Rng(int(seed).to_bytes(32, "little"))
        b = Rng(int(seed).to_bytes(32, "little"))
        assert np.array_equal(a.ternary_device(n).cpu().numpy(), b.ternary(n))
        e0, e1 = a.cbd_error_pair_device(n)
        assert np.array_equal(e0.cpu().numpy(), b.cbd_error(n))
        assert np.array_equal(e1.cpu().numpy(), b.cbd_error(n))
        assert np.array_equal(a.ternary(n), b.ternary(n))  # same state afterwards
