"""Host-side precompute (primes, CRT, sampling) and the device NTT wrapper."""

from .modmath import Modulus, ParameterError, inv_mod, is_prime, pow_mod
from .primes import gen_ntt_prime, gen_ntt_prime_chain, min_primitive_root
from .sampling import ERROR_STDDEV, Rng, fresh_seed, signed_to_residues
