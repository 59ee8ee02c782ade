"""Multi-statement fusion (FusedNode / lv.fused / salt_fused): several
assignments and a final reduction in one pass, with the results of running
the statements one after another."""

import numpy as np
import pytest
import torch

import paper_1109_1264_b200 as lv
from conftest import NP, same_bits
from oracle import restate
from paper_1109_1264_b200 import _native
from paper_1109_1264_b200.expressions import as_node

pytestmark = pytest.mark.gpu
TOL = {"f32": 1e-5, "f64": 1e-12}


def dev(v, dt):
    return lv.DenseVector.from_values(v, dt, device="cuda")


@pytest.mark.parametrize("dt", ["f32", "f64"])
def test_cg_update_one_pass_matches_sequential(dt):
    g = np.random.default_rng(21)
    for n in (1, 7, 1000, 65_537, 1 << 20):
        x, p, r, q = (g.uniform(-1, 1, n).astype(NP[dt]) for _ in range(4))
        a = 0.3125
        X, P, R, Q = (dev(v, dt) for v in (x, p, r, q))
        launches = _native.lib().salt_launch_count()
        rr = lv.fused((X, X + a * P), (R, R - a * Q), R * R)
        torch.cuda.synchronize()
        assert _native.lib().salt_launch_count() - launches == 1  # one kernel
        x1 = restate.eval_sig("L0 S0 L1 * +", [x, p], [a], dt)
        r1 = restate.eval_sig("L0 S0 L1 * -", [r, q], [a], dt)
        assert same_bits(X.to_array(), x1) and same_bits(R.to_array(), r1)
        exact = restate.exact_sum(r1 * r1)
        assert abs(float(rr) - exact) <= TOL[dt] * exact
        assert type(rr) is NP[dt]


def test_later_statements_see_earlier_assignments():
    g = np.random.default_rng(22)
    n = 50_001
    for dt in ("f32", "f64"):
        a, b, c = (g.uniform(-1, 1, n).astype(NP[dt]) for _ in range(3))
        A, B, C = (dev(v, dt) for v in (a, b, c))
        # b = a + b ; c = b * c (new b) ; b = c - b (new c, new b) ; sum(a + c)
        s = lv.fused((B, A + B), (C, B * C), (B, C - B), A + C)
        b1 = restate.eval_sig("L0 L1 +", [a, b], [], dt)
        c1 = restate.eval_sig("L0 L1 *", [b1, c], [], dt)
        b2 = restate.eval_sig("L0 L1 -", [c1, b1], [], dt)
        assert same_bits(B.to_array(), b2) and same_bits(C.to_array(), c1)
        assert same_bits(A.to_array(), a)
        exact = restate.exact_sum(restate.eval_sig("L0 L1 +", [a, c1], [], dt))
        assert abs(float(s) - exact) <= TOL[dt] * abs(exact)


def test_assign_only_fusion_and_lazy_result():
    g = np.random.default_rng(23)
    n = 100_003
    a, b = g.uniform(-1, 1, n), g.uniform(-1, 1, n)
    A, B = dev(a, "f64"), dev(b, "f64")
    D1, D2 = lv.DenseVector.zeros(n, "f64", device="cuda"), lv.DenseVector.zeros(n, "f64", device="cuda")
    assert lv.fused((D1, A + B), (D2, A - B)) is None
    assert same_bits(D1.to_array(), a + b) and same_bits(D2.to_array(), a - b)
    r = lv.fused((D1, 2.0 * D1), D1 * D2, lazy=True)
    assert isinstance(r, lv.DeviceScalar)
    d1 = 2.0 * (a + b)
    assert abs(float(r.item()) - restate.exact_sum(d1 * (a - b))) <= 1e-12 * abs(restate.exact_sum(np.abs(d1 * (a - b))))


def test_fallback_runs_statements_one_by_one():
    """CountingVector operands (not plain device vectors) take the
    statement-by-statement path: same values, the reference's traffic."""
    x = lv.CountingVector.from_values(np.arange(100.0), "f64", device="cuda")
    y = lv.CountingVector.from_values(np.ones(100), "f64", device="cuda")
    s = lv.fused((y, as_node(y) + 2.0 * as_node(x)), y * y)
    want = 1.0 + 2.0 * np.arange(100.0)
    assert y.to_values() == list(want) and s == np.sum(want * want)
    assert x.read_count == 100 and y.write_count == 100


def test_fused_update_is_faster_than_separate_passes():
    """x += a p; r -= a q; rr = r.r moves 4 reads + 2 writes once fused
    instead of 4 reads + 2 writes + 1 extra read of r in three passes."""
    n = 1 << 26
    X, P, R, Q = (lv.DenseVector.from_tensor(torch.rand(n, dtype=torch.float64, device="cuda"))
                  for _ in range(4))

    def t(fn):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(10):
            fn()
        e.record()
        e.synchronize()
        return s.elapsed_time(e) / 10

    fused = t(lambda: lv.fused((X, X + 0.5 * P), (R, R - 0.5 * Q), R * R, lazy=True))

    def separate():
        lv.axpy(0.5, P, X)
        R.assign(R - 0.5 * Q)
        lv.dot(R, R, lazy=True)

    sep = t(separate)
    assert sep / fused >= 1.15, (sep, fused)


def test_cg_example_converges():
    """examples/cg_poisson1d.py: CG on tridiag(-1, 2, -1) written with fused
    trees (matvec over shifted views, fused update) reduces the true
    residual like a plain float64 CG does."""
    import importlib.util
    from pathlib import Path

    path = Path(__file__).resolve().parents[1] / "examples" / "cg_poisson1d.py"
    spec = importlib.util.spec_from_file_location("cg_poisson1d", path)
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    n = 4096
    g = np.random.default_rng(5)
    bh = g.standard_normal(n)
    b = lv.DenseVector.from_values(bh, "f64", device="cuda")
    u, k, rel = mod.cg(b, iters=n, tol=1e-10)
    uh = u.to_array()
    au = 2 * uh
    au[1:] -= uh[:-1]
    au[:-1] -= uh[1:]
    assert np.linalg.norm(bh - au) / np.linalg.norm(bh) < 1e-8
    assert k <= n


def test_device_scalar_operands():
    """DeviceScalars scale expressions without a host round trip; results
    equal the same tree with the scalar's value passed from the host."""
    g = np.random.default_rng(31)
    n = 100_003
    for dt in ("f32", "f64"):
        x, y = (g.uniform(-1, 1, n).astype(NP[dt]) for _ in range(2))
        X, Y = dev(x, dt), dev(y, dt)
        a = lv.dot(X, Y, lazy=True)
        b = lv.dot(Y, Y, lazy=True)
        alpha = a / b  # on the device
        assert isinstance(alpha, lv.DeviceScalar)
        av, bv = a.item(), b.item()
        assert alpha.item().tobytes() == (av / bv).tobytes()  # IEEE division in dtype
        assert (-alpha).item() == -(av / bv) and (alpha * 2.0).item() == (av / bv) * NP[dt](2.0)
        assert (1.0 / alpha).item() == NP[dt](1.0) / (av / bv)
        # division by / into a host number: ONE IEEE rounding
        q = av / bv
        for c in (3.0, 7.0, 0.1, -1e-3):
            assert (alpha / c).item().tobytes() == (q / NP[dt](c)).tobytes(), c
            assert (c / alpha).item().tobytes() == (NP[dt](c) / q).tobytes(), c
        assert (alpha - b).item() == (av / bv) - bv
        D = lv.DenseVector.zeros(n, dt, device="cuda")
        launches = _native.lib().salt_launch_count()
        D.assign(alpha * X + Y)
        torch.cuda.synchronize()
        assert _native.lib().salt_launch_count() - launches == 1
        want = restate.eval_sig("S0 L0 * L1 +", [x, y], [float(alpha.item())], dt)
        assert same_bits(D.to_array(), want)
        s = lv.sum(X * alpha)  # device scalar on the right
        exact = restate.exact_sum(restate.eval_sig("S0 L0 *", [x], [float(alpha.item())], dt))
        assert abs(float(s) - exact) <= TOL[dt] * abs(exact)
        with pytest.raises(TypeError):
            lv.DeviceScalar.full(1.0, "f32" if dt == "f64" else "f64") * X  # dtype mismatch


def test_device_resident_cg_iteration_captured_in_a_graph():
    """A full CG iteration with device scalars (no host synchronisation)
    captured in a CUDA graph gives the same bits as running it eagerly."""
    import importlib.util
    from pathlib import Path

    path = Path(__file__).resolve().parents[1] / "examples" / "cg_poisson1d.py"
    spec = importlib.util.spec_from_file_location("cg_poisson1d", path)
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    n = 1 << 16
    g = np.random.default_rng(6)
    bh = g.standard_normal(n)

    def fresh():
        b = lv.DenseVector.from_values(bh, "f64", device="cuda")
        return mod.DeviceCG(b)

    eager = fresh()
    for _ in range(5):
        eager.step()
    graphed = fresh()
    graphed.step()  # warm-up outside capture (JIT, workspaces)
    graphed2 = fresh()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        graphed2.step()
    torch.cuda.current_stream().wait_stream(s)
    graphed3 = fresh()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        graphed3.step()
    for _ in range(5):
        graph.replay()
    torch.cuda.synchronize()
    assert graphed3.u.to_array().tobytes() == eager.u.to_array().tobytes()
    assert graphed3.rr.item().tobytes() == eager.rr.item().tobytes()


def test_c_fast_path_matches_python_path(monkeypatch):
    """The C host fast path (csrc/fastpath.c) takes fused statements and
    DeviceScalar operands and launches exactly what the Python path does."""
    g = np.random.default_rng(12)
    n = 70_001
    fast = _native.fastpath()
    assert fast is not None
    host = [g.uniform(-1, 1, n) for _ in range(4)]

    def run():
        x, r, p, q = (dev(h, "f64") for h in host)
        a = lv.dot(r, r, lazy=True) / lv.dot(p, q, lazy=True)
        y = lv.DenseVector.zeros(n, "f64", device="cuda")
        y.assign(a * x + p)                                   # assign with a P operand
        s1 = lv.sum(a * q, lazy=True)                         # reduce with a P operand
        s2 = lv.axpy_dot(a, x, y, r)                          # assign+reduce, P operand
        rr = lv.fused((x, x + a * p), (r, r - a * q), r * r, lazy=True)  # fused, two P operands
        lv.fused((p, r + a * p), (q, p - q))                 # fused assign-only, reads new p as D0
        return [v.to_array() for v in (x, r, p, q, y)] + [s1.item(), s2, rr.item()]

    assert fast.fused(((dev(host[0], "f64"), dev(host[1], "f64") * 2.0),), None, 0) is not None
    launches = _native.lib().salt_launch_count()
    want_fast = run()
    torch.cuda.synchronize()
    used = _native.lib().salt_launch_count() - launches
    monkeypatch.setattr(_native, "_fast", None)
    want_py = run()
    for a, b in zip(want_fast, want_py):
        assert np.asarray(a).tobytes() == np.asarray(b).tobytes()
    assert used == 2 + 1 + 1 + 1 + 1 + 1  # one kernel per statement group
    # zero length through the fast path
    e = lv.DenseVector.zeros(0, "f64", device="cuda")
    assert lv.fused((e, e * 2.0), e * e) == 0.0


def test_sharded_fused_update_with_device_scalars():
    """A CG update over ShardedVectors (here one rank) with a device-resident
    step length: one kernel per rank, the reduction's partial through the
    all-gather + fixed-order finish — same bits as the unsharded update."""
    from paper_1109_1264_b200.sharding import ShardedVector

    g = np.random.default_rng(77)
    n = 300_007
    host = [g.standard_normal(n) for _ in range(4)]

    def step(make):
        x, r, p, q = (make(h) for h in host)
        a = lv.dot(r, r, lazy=True) / lv.dot(p, q, lazy=True)
        rr = lv.fused((x, x + a * p), (r, r - a * q), r * r, lazy=True)
        lv.fused((p, r + (rr / a) * p))
        return [v.to_array() for v in (x, r, p)] + [rr.item(), a.item()]

    dense = step(lambda h: lv.DenseVector.from_values(h, "f64", device="cuda"))
    shard = step(lambda h: ShardedVector.from_global(h, "f64", device="cuda"))
    for u, v in zip(dense, shard):
        assert np.asarray(u).tobytes() == np.asarray(v).tobytes()
