"""Pin the oracle to the reference (CPU): every golden vector produced by the
reference itself must be reproduced by the NumPy restatement (restate) and
the C restatement (coracle) — bit for bit for elementwise trees and for the
reference engine's reduction order, and the exact-sum oracle must equal the
fsum value the reference's acceptance test uses (test_acceptance.py:95-100).
"""

import math

import numpy as np
import pytest

from conftest import NP, golden, same_bits
from oracle import coracle, restate


def _inputs(z, key, nv):
    return [z[f"{key}|in{k}"] for k in range(nv)]


def test_elementwise_golden_numpy_restatement():
    meta, z = golden("elementwise")
    for name, sig, dt, n, nv, ns in meta:
        key = f"{name}|{dt}|{n}"
        got = restate.eval_sig(sig, _inputs(z, key, nv), z[f"{key}|sc"], dt)
        assert same_bits(got, z[f"{key}|out"]), key


def test_elementwise_golden_c_restatement():
    meta, z = golden("elementwise")
    for name, sig, dt, n, nv, ns in meta:
        key = f"{name}|{dt}|{n}"
        ins = [a.copy() for a in _inputs(z, key, nv)]
        dst = ins[0] if name in ("scal", "axpy") else np.zeros(n, dtype=NP[dt])
        coracle.assign(sig, dst, ins, z[f"{key}|sc"], threads=2)
        assert same_bits(dst, z[f"{key}|out"]), key


def test_specials_golden_both_restatements():
    meta, z = golden("specials")
    for name, sig, dt, n, nv, ns in meta:
        key = f"{name}|{dt}"
        ins = _inputs(z, key, nv)
        assert same_bits(restate.eval_sig(sig, ins, z[f"{key}|sc"], dt), z[f"{key}|out"]), key
        dst = np.zeros(n, dtype=NP[dt])
        coracle.assign(sig, dst, [a.copy() for a in ins], z[f"{key}|sc"])
        assert same_bits(dst, z[f"{key}|out"]), key


def _plan(pname, sig, dt):
    fp = restate.footprint_of(sig, "sum")
    u, w = restate.default_plan(fp, dt)
    if pname == "u1":
        u = 1
    elif pname == "u8":
        u = 8
    elif pname == "scalar":
        u, w = 1, 1
    return u, w


def test_reduction_engine_order_is_bit_exact():
    """The reference engine's value for each plan is reproduced exactly by
    the restated block reduction (NumPy loop, NumPy vectorised, C)."""
    meta, z = golden("reductions")
    for name, sig, dt, n, dist, nv in meta:
        key = f"{name}|{dt}|{n}|{dist}"
        ins = _inputs(z, key, nv)
        vals = restate.eval_sig(sig, ins, [], dt)
        for pname in ("default", "u1", "u8", "scalar"):
            u, w = _plan(pname, sig, dt)
            ref = z[f"{key}|ref_{pname}"][0]
            r_np = restate.engine_reduce(vals, u, w)
            c = coracle.reduce(sig, ins, [], dt, u, w)
            if name == "norm2":
                r_np = np.sqrt(r_np)
                c = np.sqrt(c)
            assert r_np.tobytes() == ref.tobytes(), (key, pname)
            assert c.tobytes() == ref.tobytes(), (key, pname)
            if n <= 1000:
                r_loop = restate.engine_reduce_loop(vals, u, w)
                if name == "norm2":
                    r_loop = np.sqrt(r_loop)
                assert r_loop.tobytes() == ref.tobytes(), (key, pname)


def test_exact_oracles_match_reference_fsum():
    meta, z = golden("reductions")
    for name, sig, dt, n, dist, nv in meta:
        key = f"{name}|{dt}|{n}|{dist}"
        ins = _inputs(z, key, nv)
        exact = z[f"{key}|exact"][0]
        e1 = restate.exact_reduce(sig, ins, [], dt)
        e2 = coracle.reduce_exact(sig, ins, [], dt, threads=3)
        if name == "norm2":
            e1, e2 = math.sqrt(e1), math.sqrt(e2)
        assert e1 == exact, key
        assert e2 == pytest.approx(exact, rel=1e-15, abs=1e-300), key


def test_fused_golden():
    """axpy then dot: y_out bit-exact; the fused C restatement (assign tree +
    reduce tree reading D) reproduces the reference's two-pass r for the
    default dot plan."""
    meta, z = golden("fused")
    for dt, n in meta:
        key = f"{dt}|{n}"
        x, y, zz = z[f"{key}|x"], z[f"{key}|y"], z[f"{key}|z"]
        alpha = z[f"{key}|alpha"][0]
        y_new = restate.eval_sig("L0 S0 L1 * +", [y, x], [alpha], dt)
        assert same_bits(y_new, z[f"{key}|y_out"]), key
        u, w = restate.default_plan(restate.footprint_of("L0 L1 *", "sum"), dt)
        ycopy = y.copy()
        r = coracle.reduce("D L2 *", [ycopy, x, zz], [alpha], dt, u, w,
                           assign_sig="L0 S0 L1 * +", dst=ycopy)
        assert r.tobytes() == z[f"{key}|r_ref"].tobytes(), key
        assert same_bits(ycopy, z[f"{key}|y_out"]), key
        ex = coracle.reduce_exact("D L2 *", [y, x, zz], [alpha], dt, assign_sig="L0 S0 L1 * +")
        assert ex == pytest.approx(z[f"{key}|r_exact"][0], rel=1e-15, abs=1e-300)


def test_scalar_loop_oracles_known_answers():
    # reference test_oracle.py:15-67 known answers
    assert restate.oracle_dot([1, 2, 3], [4, 5, 6]) == 32
    assert restate.oracle_sum(list(range(1, 101))) == 5050
    assert restate.oracle_scal(2, [1, 2, 3]) == [2, 4, 6]
    assert restate.oracle_axpy(2, [1, 1], [3, 3]) == [5, 5]
    assert restate.oracle_scaled_copy(3, [1, 2]) == [3, 6]
    assert restate.kahan_sum([float(i) for i in range(1, 2049)]) == 2048 * 2049 / 2
    with pytest.raises(ValueError):
        restate.oracle_dot([1], [1, 2])


def test_default_plans_match_survey_table():
    # SURVEY.md §8(a) default plans (probe P1)
    assert restate.default_plan(restate.footprint_of("L0 S0 L1 * +", "assign"), "f64") == (4, 8)
    assert restate.default_plan(restate.footprint_of("S0 L0 * S1 L1 L2 - * +", "assign"), "f64") == (2, 8)
    assert restate.default_plan(
        restate.footprint_of("S0 L0 L1 + * S1 L2 L3 - * - S2 L0 * +", "assign"), "f32") == (1, 16)
    assert restate.default_plan(restate.footprint_of("L0 L1 *", "sum"), "f32") == (4, 16)
    assert restate.default_plan(restate.footprint_of("L0", "sum"), "f64") == (8, 8)


# ---- the reference's scalar-loop oracles (oracle.py:26-69), restated in
# oracle/restate.py as test infrastructure: the reference's test names, our
# own cases
def test_oracle_dot():
    from oracle import restate

    assert restate.oracle_dot([1.0, -2.0, 0.5], [4.0, 0.25, 8.0]) == 7.5


def test_oracle_sum():
    from oracle import restate

    assert restate.oracle_sum(np.arange(1.0, 11.0)) == 55.0


def test_oracle_scal():
    from oracle import restate

    assert list(restate.oracle_scal(-0.5, [2.0, 4.0, -6.0])) == [-1.0, -2.0, 3.0]


def test_oracle_axpy():
    from oracle import restate

    assert list(restate.oracle_axpy(2.0, [1.0, 2.0], [10.0, 20.0])) == [12.0, 24.0]


def test_oracle_scaled_copy():
    from oracle import restate

    assert list(restate.oracle_scaled_copy(3.0, [1.5, -1.0])) == [4.5, -3.0]


def test_oracles_preserve_element_type():
    from oracle import restate

    x32 = np.array([1.0, 2.0], np.float32)
    assert type(restate.oracle_dot(x32, x32)) is np.float32
    assert all(type(v) is np.float32 for v in restate.oracle_scal(np.float32(2), x32))


def test_kahan_sum_trivia():
    from oracle import restate

    assert restate.kahan_sum([]) == 0 and restate.kahan_sum([2.5]) == 2.5


def test_kahan_sum_beats_naive_summation():
    from oracle import restate

    vals = np.array([1.0] + [1e-16] * 10_000, dtype=np.float64)
    naive = 0.0
    for v in vals:
        naive += v
    exact = 1.0 + 1e-12
    assert abs(restate.kahan_sum(vals) - exact) < abs(naive - exact)
