"""Config 5: the four standard private-dataset queries over 1024 synthetic
rows on the B200, keyed and seeded like the reference PdqClient.  Every
result ciphertext must be bit-identical to the reference's run
(tests/golden/digests.json "pdq") and the decrypted answers must equal the
plaintext oracle."""

import numpy as np
import pytest

from fhe_testutil import digest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


@pytest.fixture(scope="module")
def session():
    from paper_2503_22227_b200.context import Context, PoolConfig, Scheme, params_for_profile
    from paper_2503_22227_b200.coremath.sampling import Rng
    from paper_2503_22227_b200.keys import galois_keygen, keygen, pk_gen, relin_keygen
    from paper_2503_22227_b200.pdq.columns import encode_column
    from paper_2503_22227_b200.pdq.config import PdqConfig
    from paper_2503_22227_b200.pdq.dataset import make_dataset
    from paper_2503_22227_b200.pdq.engine import LocalInverseClient, PdqEngine
    from paper_2503_22227_b200.pdq.evaluator import CkksEval, rotation_steps

    cfg = PdqConfig(base=4, digits=8, rows=1024, value_bound=1 << 16, profile="pdq")
    ctx = Context(params_for_profile("pdq", Scheme.CKKS), PoolConfig(unit_mb=64, cap_mb=2048))
    rng = Rng((1).to_bytes(32, "little"))
    sk = keygen(ctx, rng)
    pk = pk_gen(ctx, sk, rng)
    rlk = relin_keygen(ctx, sk, rng)
    gks = galois_keygen(ctx, sk, rotation_steps(ctx.n), rng)
    ev = CkksEval(ctx, rlk, gks)
    data = make_dataset(cfg, seed=20240117)
    engine = PdqEngine(ev, cfg)
    cols = {}
    for name, vals in data.items():
        col = encode_column(ev, cfg, name, vals, pk, rng)
        engine.add_column(col)
        cols[name] = col
    inv = LocalInverseClient(ev, cfg, sk, pk, rng=rng)
    return {"ctx": ctx, "sk": sk, "pk": pk, "ev": ev, "cfg": cfg, "data": data,
            "engine": engine, "cols": cols, "inv": inv, "rng": rng,
            "mask_rng": np.random.default_rng(20240118)}


def test_columns_bit_identical(session, golden):
    g = golden["pdq"]["columns"]
    for name, col in session["cols"].items():
        got = [digest(c.data.view()) for c in col.digits] + [digest(col.value.data.view())]
        assert got == g[name], name


def test_standard_queries_bit_identical(session, golden):
    from paper_2503_22227_b200.pdq.dataset import oracle_result
    from paper_2503_22227_b200.pdq.engine import (encrypt_query_constants, interpret_result,
                                                  standard_query)

    s = session
    for qid in (1, 2, 3, 4):
        g = golden["pdq"]["queries"][str(qid)]
        spec = standard_query(qid)
        temps = encrypt_query_constants(s["ev"], s["cfg"], spec, s["pk"], s["rng"])
        res = s["engine"].run(spec, channel=s["inv"], temps=temps, rng=s["mask_rng"])
        for k, c in res.cts.items():
            assert digest(c.data.view()) == g["cts"][k]["sha"], (qid, k)
            assert c.scale == g["cts"][k]["scale"] and c.level == g["cts"][k]["level"]
        got = interpret_result(s["ev"], s["sk"], res, s["cfg"].rows)
        want = oracle_result(spec, s["data"])
        if spec.agg == "index":
            assert (np.asarray(got) == want).all()
        elif spec.agg == "ratio":
            assert float(np.max(np.abs(np.asarray(got) - want))) == pytest.approx(g["max_err"])
        elif spec.agg == "sum":
            assert got == g["value"]
        else:
            assert list(got) == g["value"]
