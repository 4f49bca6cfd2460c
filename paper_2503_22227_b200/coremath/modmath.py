"""Scalar modular arithmetic on Python ints (host-side precompute only).

Same contract as the reference's coremath/modmath.py:20-136: a ``Modulus``
is an odd prime below 2^62; ``ParameterError`` signals invalid parameters.
Device kernels never call into this module.
"""

from __future__ import annotations

from dataclasses import dataclass, field


class ParameterError(ValueError):
    """Invalid numeric parameters (bad modulus, degree, level, ...)."""


# deterministic Miller-Rabin bases for n < 2^64
_BASES = (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37)


def is_prime(n: int) -> bool:
    if n < 2:
        return False
    for p in _BASES:
        if n % p == 0:
            return n == p
    d, r = n - 1, 0
    while not d & 1:
        d >>= 1
        r += 1
    bases = _BASES
    if n >= 1 << 64:
        import random

        rnd = random.Random(n)
        bases = tuple(rnd.randrange(2, n - 1) for _ in range(40))
    for a in bases:
        x = pow(a % n, d, n)
        if x in (1, n - 1):
            continue
        for _ in range(r - 1):
            x = x * x % n
            if x == n - 1:
                break
        else:
            return False
    return True


@dataclass(frozen=True)
class Modulus:
    """Odd prime modulus q < 2^62 (modmath.py:20-53)."""

    value: int
    bit_len: int = field(init=False)
    is_ntt_friendly_for: int = field(init=False)

    def __post_init__(self):
        q = self.value
        if not 2 <= q < 1 << 62:
            raise ParameterError(f"modulus {q} out of supported range [2, 2^62)")
        if q % 2 == 0:
            raise ParameterError("modulus must be odd")
        if not is_prime(q):
            raise ParameterError(f"modulus {q} is not prime")
        object.__setattr__(self, "bit_len", q.bit_length())
        two_n = 2
        while (q - 1) % (2 * two_n) == 0:
            two_n *= 2
        object.__setattr__(self, "is_ntt_friendly_for", two_n // 2)


def _val(m) -> int:
    return m.value if isinstance(m, Modulus) else int(m)


def mul_mod(a: int, b: int, m) -> int:
    return a * b % _val(m)


def add_mod(a: int, b: int, m) -> int:
    return (a + b) % _val(m)


def sub_mod(a: int, b: int, m) -> int:
    return (a - b) % _val(m)


def neg_mod(a: int, m) -> int:
    return -a % _val(m)


def pow_mod(a: int, e: int, m) -> int:
    return pow(a, e, _val(m))


def inv_mod(a: int, m) -> int:
    q = _val(m)
    if a % q == 0:
        raise ParameterError("non-invertible: 0 has no inverse")
    return pow(a, q - 2, q)
