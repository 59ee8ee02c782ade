"""Lazy DeviceScalar arithmetic compiled into the consuming kernel's scalar
program (salt_fused_prog, csrc/salt_expr.cuh load_pscalars): the same bits
as materialising the scalar with torch ops first, one launch instead of one
per scalar operation, on every path (fast/Python, interpreter, sharded)."""

import numpy as np
import pytest
import torch

import paper_1109_1264_b200 as lv
from oracle import restate
from paper_1109_1264_b200 import _native

pytestmark = pytest.mark.gpu

NP = {"f32": np.float32, "f64": np.float64}


def dev(values, dt):
    return lv.DenseVector.from_values(values, dt, device="cuda")


def scalars(dt, seed=0):
    g = np.random.default_rng([77, seed])
    return [lv.DeviceScalar.full(float(v), dt, device="cuda") for v in g.uniform(0.5, 2.0, 3)]


@pytest.mark.parametrize("dt", ["f64", "f32"])
def test_lazy_ops_are_recorded_not_launched(dt):
    a, b, c = scalars(dt)
    before = torch.cuda.memory_allocated()
    e = (a - 2.0) * b / (c + 1.5)
    f = -e + 1.0 / a
    assert e.lazy and f.lazy and f.program_size() > 5
    assert torch.cuda.memory_allocated() == before  # nothing evaluated yet
    av, bv, cv = (x.item() for x in (a, b, c))
    T = NP[dt]
    ev = (av - T(2.0)) * bv / (cv + T(1.5))
    fv = -ev + T(1.0) / av
    assert e.item().tobytes() == T(ev).tobytes() and f.item().tobytes() == T(fv).tobytes()
    assert not e.lazy  # materialised (and cached) by item()


@pytest.mark.parametrize("dt", ["f64", "f32"])
def test_cg_update_with_a_lazy_step_length_is_one_launch(dt):
    """x += alpha*p; r -= alpha*q; rr = r.r with alpha = rr0 / pq — the
    division runs in the fused kernel's prologue: ONE libsalt launch, the
    lazy scalar never materialised, and the bits of the eager path."""
    n = 300_007
    g = np.random.default_rng(5)
    xv, pv, rv, qv = (g.standard_normal(n).astype(NP[dt]) for _ in range(4))
    X, P, R, Q = (dev(v, dt) for v in (xv, pv, rv, qv))
    rr0 = lv.dot(R, R, lazy=True)
    pq = lv.dot(P, Q, lazy=True)
    alpha = rr0 / pq
    assert alpha.lazy
    lib = _native.lib()
    torch.cuda.synchronize()
    l0 = lib.salt_launch_count()
    rr = lv.fused((X, X + alpha * P), (R, R - alpha * Q), R * R, lazy=True)
    torch.cuda.synchronize()
    assert lib.salt_launch_count() - l0 == 1
    assert alpha.lazy  # compiled into the kernel, never evaluated on its own
    # eager reference: the same update with alpha materialised first
    X2, P2, R2, Q2 = (dev(v, dt) for v in (xv, pv, rv, qv))
    a_val = (rr0.item() / pq.item())
    rr_eager = lv.fused((X2, X2 + lv.DeviceScalar.full(a_val, dt, device="cuda") * P2),
                        (R2, R2 - lv.DeviceScalar.full(a_val, dt, device="cuda") * Q2), R2 * R2, lazy=True)
    assert X.to_array().tobytes() == X2.to_array().tobytes()
    assert R.to_array().tobytes() == R2.to_array().tobytes()
    assert rr.item().tobytes() == rr_eager.item().tobytes()
    # and against the oracle, with alpha = the IEEE quotient in dtype
    x_new = restate.eval_sig("L0 S0 L1 * +", [xv, pv], [float(a_val)], dt)
    assert X.to_array().tobytes() == x_new.tobytes()


@pytest.mark.parametrize("dt", ["f64", "f32"])
def test_program_shapes_match_materialised_scalars(dt):
    n = 100_003
    g = np.random.default_rng(9)
    xv, yv = (g.uniform(-1, 1, n).astype(NP[dt]) for _ in range(2))
    a, b, c = scalars(dt, 3)
    cases = [
        lambda: a / b,
        lambda: -(a * b) + c,
        lambda: 3.0 - a,
        lambda: 1.0 / a,
        lambda: (a + 0.25) * (b - c) / (a * c),
        lambda: a / b / c / a / b,
    ]
    for make in cases:
        s_lazy, s_eager = make(), make()
        s_eager.tensor  # materialise with torch ops
        Y1, Y2 = dev(yv, dt), dev(yv, dt)
        X = dev(xv, dt)
        Y1.assign(Y1 + s_lazy * X)           # scalar program (Python path)
        Y2.assign(Y2 + s_eager * X)          # raw device scalar (C fast path)
        assert Y1.to_array().tobytes() == Y2.to_array().tobytes()
        want = restate.eval_sig("L0 S0 L1 * +", [yv, xv], [float(s_eager.item())], dt)
        assert Y1.to_array().tobytes() == want.tobytes()
        r1 = lv.dot(X, s_lazy * X)
        r2 = lv.dot(X, s_eager * X)
        assert np.asarray(r1).tobytes() == np.asarray(r2).tobytes()


def test_two_lazy_scalars_share_raw_operands_and_host_constants():
    n = 50_000
    g = np.random.default_rng(4)
    xv, yv, zv = (g.standard_normal(n) for _ in range(3))
    X, Y, Z = (dev(v, "f64") for v in (xv, yv, zv))
    a, b, _ = scalars("f64", 1)
    s1, s2 = a / b, (a - 0.5) * 2.0
    W = lv.DenseVector.zeros(n, "f64", device="cuda")
    W.assign(1.5 * X + s1 * (Y - s2 * Z))
    t1, t2 = float(s1.item()), float(s2.item())
    want = restate.eval_sig("S0 L0 * S1 L1 S2 L2 * - * +", [xv, yv, zv], [1.5, t1, t2], "f64")
    assert W.to_array().tobytes() == want.tobytes()


def test_oversized_program_is_materialised():
    a, b, _ = scalars("f64", 2)
    s = a
    for i in range(30):  # > MAX_PROGRAM_OPS operations
        s = s * 1.0000001 + b
    n = 4096
    xv = np.linspace(-1, 1, n)
    X, Y = dev(xv, "f64"), lv.DenseVector.zeros(n, "f64", device="cuda")
    Y.assign(s * X)
    want = restate.eval_sig("S0 L0 *", [xv], [float(s.item())], "f64")
    assert Y.to_array().tobytes() == want.tobytes()


def test_interpreter_runs_the_same_program():
    lib = _native.lib()
    n = 70_001
    g = np.random.default_rng(8)
    xv, yv = (g.standard_normal(n) for _ in range(2))
    a, b, c = scalars("f64", 6)
    outs = []
    for interp in (0, 1):
        lib.salt_set_force_interp(interp)
        try:
            X, Y = dev(xv, "f64"), dev(yv, "f64")
            s = (a - c) / b
            r = lv.fused((Y, Y - s * X), Y * X)
            outs.append((Y.to_array().tobytes(), np.asarray(r).tobytes()))
        finally:
            lib.salt_set_force_interp(0)
    assert outs[0] == outs[1]


def test_sharded_vectors_with_a_lazy_scalar():
    """ShardedVector (world 1, no process group): the exchange-capable
    reduction path passes the program too."""
    n = 40_000
    g = np.random.default_rng(10)
    xv, yv = (g.standard_normal(n) for _ in range(2))
    X = lv.ShardedVector.from_global(xv, "f64", device="cuda")
    Y = lv.ShardedVector.from_global(yv, "f64", device="cuda")
    a, b, _ = scalars("f64", 7)
    s = a / b
    r = lv.fused((Y, Y + s * X), Y * Y)
    y_new = restate.eval_sig("L0 S0 L1 * +", [yv, xv], [float(s.item())], "f64")
    assert Y.local.to_array().tobytes() == y_new.tobytes()
    ex = restate.exact_sum(y_new * y_new)
    assert abs(float(r) - ex) <= 1e-12 * ex


def test_lazy_scalar_refuses_an_operand_modified_in_place():
    """copy_ into an operand after recording would silently change the
    value a lazy scalar stands for: it raises instead."""
    a, b, _ = scalars("f64", 11)
    s = a / b
    b.copy_(3.0)
    with pytest.raises(RuntimeError, match="modified in place"):
        s.item()
    X = dev(np.ones(64), "f64")
    t = a * 2.0
    a.copy_(1.0)
    with pytest.raises(RuntimeError, match="modified in place"):
        X.assign(X + t * X)
    # materialised before the copy_: keeps the old value (eager semantics)
    u = a + 1.0
    u.tensor
    a.copy_(5.0)
    assert u.item() == 2.0


def test_c_fast_path_compiles_lazy_scalars(monkeypatch):
    """The CPython fast path builds the scalar program itself (no Python
    lowering, no torch launch): runtime.run_fused is never reached."""
    from paper_1109_1264_b200 import runtime

    def boom(*a, **k):
        raise AssertionError("Python path taken")

    n = 10_000
    g = np.random.default_rng(12)
    xv, yv = (g.standard_normal(n) for _ in range(2))
    X, Y = dev(xv, "f64"), dev(yv, "f64")
    a, b, c = scalars("f64", 13)
    monkeypatch.setattr(runtime, "run_fused", boom)
    s = (a - 0.5) / b + c
    r = lv.fused((Y, Y + s * X), Y * X)                 # fused assign + reduce
    Y.assign(Y - (a / c) * X)                           # plain assign with a lazy alpha
    r2 = lv.dot(X, (b * 2.0) * Y)                       # reduce with a lazy alpha
    assert s.lazy
    monkeypatch.undo()
    sv, acv, b2 = float(s.item()), float((a / c).item()), float((b * 2.0).item())
    y1 = restate.eval_sig("L0 S0 L1 * +", [yv, xv], [sv], "f64")
    y2 = restate.eval_sig("L0 S0 L1 * -", [y1, xv], [acv], "f64")
    assert Y.to_array().tobytes() == y2.tobytes()
    ex = restate.exact_sum(y1 * xv)
    assert abs(float(r) - ex) <= 1e-12 * abs(ex)
    ex2 = restate.exact_sum(xv * (b2 * y2))
    assert abs(float(r2) - ex2) <= 1e-12 * abs(ex2)
