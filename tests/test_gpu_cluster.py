"""Small-n reductions can run as ONE thread-block cluster (<= 16 CTAs) whose
partials meet in distributed shared memory (the default for 3-32 tiles
until the collector took over every grid of 3+ tiles; SALT_COLLECT_MIN=33
restores it, which is how this test reaches it).  The fold order is the ticket
path's (thread t takes CTA t, then the same block tree), so forcing the
ticket combine on the same grid (SALT_CLUSTER_COMBINE=0) gives the same
bits; and the values stay within the reduction tolerance of the oracle."""

import json
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

from oracle import restate

ROOT = Path(__file__).resolve().parents[1]

SCRIPT = r"""
import json, sys
import numpy as np
sys.path.insert(0, sys.argv[1])
import paper_1109_1264_b200 as lv
out = {}
for n in (5000, 16387, 65536, 131067, 262144):
    g = np.random.default_rng(n)
    x, y, z = (g.standard_normal(n) for _ in range(3))
    X, Y, Z = (lv.DenseVector.from_values(v, "f64", device="cuda") for v in (x, y, z))
    Xs, Ys = (lv.DenseVector.from_values(v, "f32", device="cuda") for v in (x, y))
    out[n] = [float(lv.dot(X, Y)).hex(), float(lv.norm2(X)).hex(), float(lv.dot(Xs, Ys)).hex(),
              float(lv.axpy_dot(0.5, X, Y, Z)).hex()]
print(json.dumps(out))
"""


def run(env_extra):
    env = dict(os.environ, **env_extra)
    r = subprocess.run([sys.executable, "-c", SCRIPT, str(ROOT)], capture_output=True, text=True,
                       env=env, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


@pytest.mark.gpu
def test_cluster_combine_matches_ticket_combine_and_oracle():
    a = run({"SALT_COLLECT_MIN": "33"})
    b = run({"SALT_COLLECT_MIN": "33", "SALT_CLUSTER_COMBINE": "0"})
    assert a == b
    # the default route for these sizes (the collector) agrees to a rounding
    c = run({})
    for n in a:
        for va, vc in zip(a[n], c[n]):
            va, vc = float.fromhex(va), float.fromhex(vc)
            assert abs(va - vc) <= 2.3e-16 * abs(va) or abs(va - vc) <= 1.2e-7 * abs(va) and va == np.float32(va)
    for n, vals in a.items():
        n = int(n)
        g = np.random.default_rng(n)
        x, y, z = (g.standard_normal(n) for _ in range(3))
        dot, nrm, sdot, ad = (float.fromhex(v) for v in vals)
        assert abs(dot - restate.exact_sum(x * y)) <= 1e-12 * abs(restate.exact_sum(x * y)) + 1e-300
        want = np.sqrt(restate.exact_sum(x * x))
        assert abs(nrm - want) <= 1e-12 * want
        xs, ys = x.astype(np.float32), y.astype(np.float32)
        ws = restate.exact_sum((xs * ys).astype(np.float64))
        assert abs(sdot - ws) <= 1e-5 * abs(ws)
        y2 = y + 0.5 * x
        wa = restate.exact_sum(y2 * z)
        assert abs(ad - wa) <= 1e-12 * abs(wa)
