"""The opt-in one-pass cluster NTT (csrc/ntt_cluster.cuh, FHE_NTT_CLUSTER=1)
is bit-identical to the C oracle restatement of the reference transform
(coremath/_kernels.py:35-99) and is the path that ran."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


def test_cluster_ntt_matches_oracle():
    env = dict(os.environ, FHE_NTT_CLUSTER="1")
    res = subprocess.run([sys.executable, os.path.join(HERE, "helpers", "cluster_ntt_parity.py")],
                         env=env, capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stderr[-2000:]
    got = json.loads(res.stdout.strip().splitlines()[-1])
    assert got, "no cases ran"
    for case, r in got.items():
        assert r["cluster_launches"] == 1, (case, r)
        assert r["bad_rows"] == 0, (case, r)
