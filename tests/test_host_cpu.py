"""Host-side logic and the C-ABI boundary, without a GPU."""

import ctypes
import json
import os
import re

import numpy as np
import pytest

from fhe_testutil import GOLDEN, ROOT

HEADER = os.path.join(ROOT, "include", "fhe_sm100.h")


def test_library_exports_every_header_symbol():
    from paper_2503_22227_b200 import _native

    lib = _native.load_library()
    declared = set(re.findall(r"\b(fhe_\w+)\s*\(", open(HEADER).read()))
    assert declared, "no declarations parsed"
    for name in declared:
        assert hasattr(lib, name), name
    assert declared == set(_native.SIGNATURES), declared ^ set(_native.SIGNATURES)


def test_compute_path_fails_loudly_without_gpu():
    import torch

    from paper_2503_22227_b200 import _native
    from paper_2503_22227_b200.context import Context, params_for_profile

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(_native.NativeUnavailable):
        _native.lib()
    with pytest.raises(_native.NativeUnavailable):
        Context(params_for_profile("desk4k", "ckks"))


def test_library_is_sm100a():
    lib = os.path.join(ROOT, "paper_2503_22227_b200", "lib", "libfhe_sm100.so")
    out = os.popen(f"cuobjdump -lelf {lib} 2>&1").read()
    assert "sm_100a" in out, out[:500]


def test_validation_mirrors_reference():
    from paper_2503_22227_b200.context import EncryptionParams, Scheme
    from paper_2503_22227_b200.coremath.primes import gen_ntt_prime_chain

    qs = tuple(m.value for m in gen_ntt_prime_chain(36, 64, 3))
    assert EncryptionParams(Scheme.CKKS, 64, qs, default_scale=2.0 ** 30).validate() == []
    causes = EncryptionParams(Scheme.CKKS, 63, qs + qs[:1]).validate()
    assert any("power of two" in c for c in causes)
    assert any("not distinct" in c for c in causes)
    assert any("default scale" in c for c in causes)
    assert any("plain modulus" in c for c in EncryptionParams(Scheme.BFV, 64, qs).validate())
    long = tuple(m.value for m in gen_ntt_prime_chain(40, 64, 18))
    assert any("chain length 18" in c for c in EncryptionParams(Scheme.CKKS, 64, long,
                                                                  default_scale=1.0).validate())
    # hybrid parameters lift the chain cap and check the special primes
    ps = tuple(m.value for m in gen_ntt_prime_chain(40, 64, 2, extra_exclude=long))
    ok = EncryptionParams(Scheme.CKKS, 64, long, default_scale=1.0, special_moduli=ps,
                          ks_alpha=6)
    assert ok.validate() == [] and ok.dnum == 3
    bad = EncryptionParams(Scheme.CKKS, 64, long, default_scale=1.0, ks_alpha=2)
    assert any("special moduli" in c for c in bad.validate())


@pytest.mark.parametrize("profile,n,levels", [("desk4k", 4096, 3), ("desk8k", 8192, 6),
                                              ("pdq", 4096, 13), ("big32k", 32768, 16)])
def test_profiles(profile, n, levels):
    from paper_2503_22227_b200.context import params_for_profile

    p = params_for_profile(profile, "ckks")
    assert p.n == n and p.level_count == levels and p.validate() == []


def test_primes_and_roots_match_oracle():
    from oracle import rns_oracle as orc
    from paper_2503_22227_b200.coremath.primes import gen_ntt_prime_chain, min_primitive_root

    for bits, n, c in ((36, 64, 3), (50, 1 << 16, 4), (60, 1 << 16, 2)):
        ours = [m.value for m in gen_ntt_prime_chain(bits, n, c)]
        assert ours == orc.prime_chain(bits, n, c)
    for q in orc.prime_chain(40, 256, 3):
        assert min_primitive_root(q, 512) == orc.min_root(q, 512)


def test_galois_permutation_host_copy():
    from oracle import rns_oracle as orc
    from paper_2503_22227_b200.coremath.ntt import exponent_map

    n = 256
    exps = exponent_map(n)
    assert sorted(((exps - 1) // 2).tolist()) == list(range(n))
    pos = np.empty(2 * n, dtype=np.int64)
    pos[exps] = np.arange(n)
    for elt in (5, 25, 2 * n - 1):
        assert (pos[(exps * elt) % (2 * n)] == orc.galois_perm(n, elt)).all()


def test_crt_against_python_ints():
    from paper_2503_22227_b200.coremath.crt import (RnsBase, crt_reconstruct,
                                                    crt_reconstruct_centered,
                                                    crt_reconstruct_poly)
    from paper_2503_22227_b200.coremath.primes import gen_ntt_prime_chain

    base = RnsBase(gen_ntt_prime_chain(45, 64, 4))
    rng = np.random.default_rng(3)
    xs = [int(v) for v in rng.integers(0, 1 << 62, 8)]
    xs = [x * 12345678901 % base.product for x in xs]
    rows = np.array([[x % q for x in xs] for q in base.values], dtype=np.uint64)
    assert crt_reconstruct_poly(rows, base) == xs
    assert crt_reconstruct(rows[:, 0], base) == xs[0]
    c = crt_reconstruct_centered(base.residues_of(base.product - 5), base)
    assert c == -5


def test_sampler_replays_reference_stream(golden_arrays):
    """The host sampler reproduces the reference's secret key coefficients
    (config 1, seed 1) exactly."""
    from fhe_testutil import seeded_rng

    assert (seeded_rng(1).ternary(8192) == golden_arrays["ckks_c1"]["sk_coeffs"]).all()


def test_ckks_embedding_round_trip():
    from paper_2503_22227_b200.schemes.ckks import embed_forward, embed_inverse

    rng = np.random.default_rng(1)
    v = rng.uniform(-1, 1, 512) + 1j * rng.uniform(-1, 1, 512)
    assert np.allclose(embed_forward(embed_inverse(v, 1024), 1024), v, atol=1e-12)


@pytest.mark.parametrize("p", [2, 3, 4, 5])
def test_compare_interpolants_truth_tables(p):
    from paper_2503_22227_b200.pdq.compare import lt_coeffs

    w = np.exp(2j * np.pi / p)
    c = lt_coeffs(p)
    for a in range(p):
        for b in range(p):
            z, y = w ** a, w ** b
            eq = (1 + sum(z ** t * y ** (p - t) for t in range(1, p))) / p
            lt = sum(c[t, s] * z ** t * y ** s for t in range(p) for s in range(p))
            assert abs(eq - (a == b)) < 1e-9
            assert abs(lt - (a < b)) < 1e-9


def test_query_specs_and_digits():
    from paper_2503_22227_b200.pdq.config import digit_decompose, digit_recompose
    from paper_2503_22227_b200.pdq.engine import QuerySpec, predicate_atoms, standard_query

    for v in (0, 1, 17, 65535):
        assert digit_recompose(digit_decompose(v, 4, 8), 4) == v
    for q in (1, 2, 3, 4):
        spec = standard_query(q)
        assert QuerySpec.from_json(spec.to_json()) == spec
    assert [a.op for a in predicate_atoms(standard_query(1).predicate)] == ["<=", "!="]


def test_pdq_plaintext_oracle_matches_reference_index(golden):
    from paper_2503_22227_b200.pdq.config import PdqConfig
    from paper_2503_22227_b200.pdq.dataset import make_dataset, oracle_result
    from paper_2503_22227_b200.pdq.engine import standard_query

    data = make_dataset(PdqConfig(), seed=20240117)
    mask = oracle_result(standard_query(1), data)
    assert mask.astype(int).tolist() == golden["pdq"]["queries"]["1"]["value"]
    assert oracle_result(standard_query(2), data) == golden["pdq"]["queries"]["2"]["oracle"]


def test_kernel_seam_signatures_match_reference():
    """The seam module mirrors rnsfhe.coremath._kernels (_kernels.py:86-173):
    same names and positional parameters (it imports without a GPU)."""
    import inspect

    from paper_2503_22227_b200.coremath import _kernels

    want = {
        "ntt_batch": ["a", "psi", "psi_sh", "q", "mod_idx"],
        "intt_batch": ["a", "ipsi", "ipsi_sh", "n_inv", "n_inv_sh", "q", "mod_idx"],
        "mul_batch": ["a", "b", "out", "q", "qinv", "r2", "mod_idx"],
        "neg_mul_batch": ["a", "b", "out", "q", "qinv", "r2", "mod_idx"],
        "mul_add_batch": ["a", "b", "c", "out", "q", "qinv", "r2", "mod_idx"],
    }
    for name, params in want.items():
        assert list(inspect.signature(getattr(_kernels, name)).parameters) == params, name
