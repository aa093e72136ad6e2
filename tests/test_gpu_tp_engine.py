"""Tensor-parallel and hybrid partitions through the persistent decode engine with the
TP merges inside it ("merged twice", Table 4), run as
concurrent streams on ONE GPU with in-process communicators (if_comm_create_local:
each rank's engine gets SMs / devices CTAs, so the ranks of a group are co-resident).
Each case runs in a subprocess (scripts/tp_engine_check.py): several autoregressive
steps against the oracle's unpartitioned fp64 stack at 1e-3 normwise, bit-identical
outputs on every TP rank (fixed rank-order sums), and one engine launch per rank per
step (plus the stage hand-off kernels) instead of ~10 launches per layer.
"""
import json
import os
import subprocess
import sys

import pytest

from gpu_util import dev

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(mode):
    dev()
    r = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "tp_engine_check.py"), mode, "3"],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


@pytest.mark.parametrize("mode,launches", [("tensor", 2), ("tensor4", 4), ("hybrid", 8), ("layer", 4)])
def test_engine_partitioned_decode_vs_oracle(mode, launches):
    res = _run(mode)
    print(res)
    assert max(res["errs"]) <= 1e-3, res
    assert res["bitwise_equal_tp"], res
    # TP: one engine launch per rank; by_layer / hybrid: + one send on each non-last rank
    # and one recv on each non-first rank
    assert all(n == launches for n in res["launches_per_step"]), res
