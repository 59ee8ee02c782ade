"""The collector combine (csrc/salt_expr.cuh collect_epilogue) at the sizes
where the launch geometry changes, with special values, and against the
round-1 ticket combine (SALT_COMBINE=ticket, a separate process): every
result within one rounding of the exact sum, deterministic, and the
reference's inf / NaN semantics."""

import json
import os
import subprocess
import sys

import numpy as np
import pytest

import paper_1109_1264_b200 as lv
from conftest import ROOT
from oracle import restate

pytestmark = pytest.mark.gpu

# f64 dot: 512-element vectors x UNR 2 per tile -> tiles = ceil(n / 2048);
# 3+ tiles take the collector (one streaming CTA per tile; 1 collector warp
# below 128 streaming CTAs, 2 below 8,192, 4 beyond); > 65,536 tiles grow the
# tiles per CTA.  Streaming-CTA counts on both sides of every boundary, and
# counts that leave the collector's warps partly filled.
SIZES = [2048 * 2 + 1, 2048 * 3, 2048 * 5 - 7, 2048 * 31 + 3, 2048 * 32, 2048 * 32 + 1, 2048 * 33 + 5,
         2048 * 127, 2048 * 127 + 1, 2048 * 128 + 9, 2048 * 510, 2048 * 511 + 7, (1 << 22) + 3,
         2048 * 8191, 2048 * 8191 + 5, 2048 * 8192 + 1, (1 << 24) - 5, 2048 * 65536 + 2048 * 3 + 1]


def _vals(n, seed):
    return np.random.default_rng([5, seed, n % 100003]).standard_normal(n)


@pytest.mark.parametrize("n", SIZES)
def test_collector_sizes_are_exact_to_a_rounding_and_deterministic(n):
    x, y = _vals(n, 1), _vals(n, 2)
    X, Y = (lv.DenseVector.from_values(v, "f64", device="cuda") for v in (x, y))
    r = [lv.dot(X, Y) for _ in range(3)]
    assert len({np.float64(v).tobytes() for v in r}) == 1
    ex = restate.exact_sum(x * y)
    assert abs(float(r[0]) - ex) <= 2.3e-16 * abs(ex) + 1e-300
    q = lv.norm2(X)
    exq = np.sqrt(restate.exact_sum(x * x))
    assert abs(float(q) - exq) <= 2.3e-16 * exq


@pytest.mark.parametrize("special", ["inf", "-inf", "nan", "inf-inf"])
@pytest.mark.parametrize("n", [2048 * 5 + 3, 1 << 21])  # 6 and 1,024 streaming CTAs
def test_collector_special_values(special, n):
    x = _vals(n, 3)
    where = [17, n // 3, n - 2]  # in the first, a middle and the last streaming CTA
    if special == "inf":
        x[where[1]] = np.inf
    elif special == "-inf":
        x[where[2]] = -np.inf
    elif special == "nan":
        x[where[0]] = np.nan
    else:
        x[where[0]], x[where[2]] = np.inf, -np.inf
    X = lv.DenseVector.from_values(x, "f64", device="cuda")
    got = float(lv.sum(X))
    want = float(np.sum(x))  # inf, -inf or NaN: the plain IEEE sum's result
    assert (np.isnan(got) and np.isnan(want)) or got == want, (got, want)


_SCRIPT = r"""
import json, sys
import numpy as np
sys.path.insert(0, sys.argv[1])
import paper_1109_1264_b200 as lv
out = {}
for n in map(int, sys.argv[2].split(",")):
    g = np.random.default_rng([5, 9, n])
    x, y = g.standard_normal(n), g.standard_normal(n)
    X, Y = (lv.DenseVector.from_values(v, "f64", device="cuda") for v in (x, y))
    out[n] = [float(lv.dot(X, Y)).hex(), float(lv.norm2(X)).hex()]
print(json.dumps(out))
"""


def test_collector_and_ticket_combines_agree_to_a_rounding():
    sizes = [2048 * 7 + 1, 2048 * 40, 2048 * 600, (1 << 23) + 11]
    res = {}
    for combine in ("collector", "ticket"):
        env = dict(os.environ)
        if combine == "ticket":
            env["SALT_COMBINE"] = "ticket"
        else:
            env.pop("SALT_COMBINE", None)
        r = subprocess.run([sys.executable, "-c", _SCRIPT, str(ROOT), ",".join(map(str, sizes))],
                           capture_output=True, text=True, env=env, timeout=600, check=True)
        res[combine] = json.loads(r.stdout.strip().splitlines()[-1])
    for n in sizes:
        for k in range(2):
            a = float.fromhex(res["collector"][str(n)][k])
            b = float.fromhex(res["ticket"][str(n)][k])
            assert abs(a - b) <= 4.5e-16 * abs(b), (n, k, a, b)


def test_collector_warp_counts_agree_to_a_rounding():
    """1 / 2 / 4 / 8 collector warps change the fold order (the product picks
    1 / 2 / 4 by grid size), never the value beyond a rounding."""
    sizes = [2048 * 5 + 1, 2048 * 200 + 3, (1 << 23) + 11]
    res = {}
    for w in ("1", "2", "4", "8"):
        env = dict(os.environ, SALT_COLLECT_WARPS=w)
        r = subprocess.run([sys.executable, "-c", _SCRIPT, str(ROOT), ",".join(map(str, sizes))],
                           capture_output=True, text=True, env=env, timeout=600, check=True)
        res[w] = json.loads(r.stdout.strip().splitlines()[-1])
    for n in sizes:
        for k in range(2):
            vals = [float.fromhex(res[w][str(n)][k]) for w in res]
            assert max(vals) - min(vals) <= 4.5e-16 * abs(vals[0]), (n, k, vals)
