"""Multi-GPU layouts of the private-dataset query, run as
two processes on the leased GPU over gloo (the bench runs them over NCCL,
one GPU per rank):

* the (atom, digit) unit split of the real PdqEngine at world 2 gives result
  ciphertexts bit-identical to the reference's run (tests/golden "pdq");
* the row-batch layout (4 blocks of N/2 rows) gives the same aggregate words
  at world 1 and world 2 (all-reduce + mod-q fix-up == ckks_add over all
  blocks), and the decrypted sum / average match the plaintext oracle.
"""
import json
import os
import socket
import sys

import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "helpers"))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _spawn(fn, world, *args):
    import torch.multiprocessing as mp

    out = mp.Manager().dict()
    mp.spawn(fn, args=(world, _port(), out) + args, nprocs=world, join=True)
    return {r: json.loads(out[r]) for r in range(world)}


def test_unit_sharded_engine_world2_matches_reference(golden):
    import pdq_workers

    got = _spawn(pdq_workers.units_worker, 2)
    for rank in (0, 1):
        for qid in ("1", "2", "3", "4"):
            want = golden["pdq"]["queries"][qid]["cts"]
            for k, (sha, scale, level) in got[rank][qid].items():
                assert sha == want[k]["sha"], (rank, qid, k)
                assert scale == want[k]["scale"] and level == want[k]["level"]


def test_rowblocks_world2_equals_world1():
    import numpy as np

    import pdq_workers
    from paper_2503_22227_b200.pdq.config import PdqConfig
    from paper_2503_22227_b200.pdq.dataset import make_dataset, oracle_result
    from paper_2503_22227_b200.pdq.engine import standard_query

    rows = 4 * 2048
    one = _spawn(pdq_workers.rowblocks_worker, 1)[0]
    two = _spawn(pdq_workers.rowblocks_worker, 2)
    assert sorted(two[0]["blocks"] + two[1]["blocks"]) == [0, 1, 2, 3]
    for qid in ("2", "4"):
        for rank in (0, 1):
            assert two[rank][qid] == one[qid], (qid, rank)
    data = make_dataset(PdqConfig(rows=rows), seed=20240117)
    want_sum = oracle_result(standard_query(2), data)
    assert abs(one["2_dec"]["sum"] - want_sum) < 1e-3 * max(1.0, abs(want_sum))
    empty, want_avg = oracle_result(standard_query(4), data)
    assert not empty
    assert two[0]["4_dec"]["avg"] == pytest.approx(want_avg, rel=1e-3)
    assert np.isclose(two[0]["4_dec"]["count"],
                      float((data["b"] <= data["c"]).__and__(data["d"] == data["e"]).sum()),
                      atol=1e-2)
