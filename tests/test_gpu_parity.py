"""GPU parity against the reference's golden vectors and the oracle.

Every evaluation here goes through the public API (DenseVector / ops /
execute_*) and therefore through libsalt.so's C ABI; the oracle and the
golden fixtures (produced by the reference itself) are only the checkers.
Bar: bit-exact for elementwise trees; for reductions |r - exact| <=
tol * |exact| with tol = 1e-12 (f64) / 1e-5 (f32) (BASELINE.json north_star).
"""

import numpy as np
import pytest
import torch

import paper_1109_1264_b200 as lv
from conftest import NP, golden, same_bits
from oracle import restate
from paper_1109_1264_b200 import _native
from paper_1109_1264_b200.engine import execute_reduce
from paper_1109_1264_b200.expressions import AssignNode, AssignReduceNode, ScaleNode, SumNode, as_node

pytestmark = pytest.mark.gpu

TOL = {"f32": 1e-5, "f64": 1e-12}


def dev(values, dt):
    return lv.DenseVector.from_values(values, dt, device="cuda")


def _build(name, v, s, d):
    """The same API calls make_golden.py made on the reference."""
    if name == "copy":
        d.assign(v[0])
    elif name == "scaled_copy":
        lv.scaled_copy(s[0], v[0], d)
    elif name == "t1":
        d.assign(v[0] + (v[1] - v[2]))
    elif name == "t2":
        d.assign(s[0] * v[0] + s[1] * (v[1] - v[2]))
    elif name == "etree":
        d.assign(s[0] * (v[0] + v[1]) - s[1] * (v[2] - v[3]) + s[2] * v[0])
    elif name == "mul3":
        d.assign(v[0] * v[1] * v[2])
    elif name == "neg_sum":
        d.assign(-(v[0] + v[1]))
    elif name == "mixed":
        d.assign((v[0] * v[1] - v[2] * v[0]) + s[0] * v[1])
    elif name == "scale_right":
        d.assign((v[0] - v[1]) * s[0])
    else:
        raise AssertionError(name)


def test_elementwise_golden_bit_exact():
    meta, z = golden("elementwise")
    for name, sig, dt, n, nv, ns in meta:
        key = f"{name}|{dt}|{n}"
        ins = [z[f"{key}|in{k}"] for k in range(nv)]
        sc = [float(x) for x in z[f"{key}|sc"]]
        vecs = [dev(a, dt) for a in ins]
        if name == "scal":
            lv.scal(sc[0], vecs[0])
            got = vecs[0].to_array()
        elif name == "axpy":
            lv.axpy(sc[0], vecs[1], vecs[0])
            got = vecs[0].to_array()
        else:
            d = lv.DenseVector.zeros(n, dt, device="cuda")
            _build(name, vecs, sc, d)
            got = d.to_array()
        assert same_bits(got, z[f"{key}|out"]), key


def test_specials_bit_exact():
    """inf, nan, signed zeros, subnormals, max values (no FTZ, no FMA)."""
    meta, z = golden("specials")
    for name, sig, dt, n, nv, ns in meta:
        key = f"{name}|{dt}"
        vecs = [dev(z[f"{key}|in{k}"], dt) for k in range(nv)]
        d = lv.DenseVector.zeros(n, dt, device="cuda")
        _build(name, vecs, [float(x) for x in z[f"{key}|sc"]], d)
        assert same_bits(d.to_array(), z[f"{key}|out"]), key


def _red(name, vecs, **kw):
    if name == "dot":
        return lv.dot(vecs[0], vecs[1], **kw)
    if name == "sum":
        return lv.sum(vecs[0], **kw)
    if name == "norm2":
        return lv.norm2(vecs[0], **kw)
    return execute_reduce(SumNode(as_node(vecs[0]) + (as_node(vecs[1]) - as_node(vecs[2]))), **kw)


def test_reductions_golden_within_tolerance_of_exact():
    meta, z = golden("reductions")
    for name, sig, dt, n, dist, nv in meta:
        key = f"{name}|{dt}|{n}|{dist}"
        vecs = [dev(z[f"{key}|in{k}"], dt) for k in range(nv)]
        got = _red(name, vecs)
        assert type(got) is NP[dt], key
        exact = z[f"{key}|exact"][0]
        if exact == 0.0:
            assert float(got) == 0.0, key
            continue
        err = abs(float(got) - exact) / abs(exact)
        # the GPU sum is double-double then rounded once to the element type
        assert err <= TOL[dt], (key, err)
        assert err <= np.finfo(NP[dt]).eps, (key, err)


def test_reductions_ignore_plan_options_and_are_deterministic():
    meta, z = golden("reductions")
    for name, sig, dt, n, dist, nv in meta[::7]:
        key = f"{name}|{dt}|{n}|{dist}"
        vecs = [dev(z[f"{key}|in{k}"], dt) for k in range(nv)]
        base = _red(name, vecs)
        for opts in ({"unroll": 1}, {"unroll": 8, "packages": 2}, {"stepped": True},
                     {"backend": lv.scalar_backend(dt)}):
            assert _red(name, vecs, **opts).tobytes() == base.tobytes(), (key, opts)


def test_fused_axpy_dot_golden():
    meta, z = golden("fused")
    for dt, n in meta:
        key = f"{dt}|{n}"
        X, Y, Z = (dev(z[f"{key}|{k}"], dt) for k in "xyz")
        r = lv.axpy_dot(float(z[f"{key}|alpha"][0]), X, Y, Z)
        assert same_bits(Y.to_array(), z[f"{key}|y_out"]), key
        exact = z[f"{key}|r_exact"][0]
        if exact != 0.0:
            assert abs(float(r) - exact) <= TOL[dt] * abs(exact), key


def test_known_answers():
    # reference test_ops.py / test_engine.py known answers
    for dt in ("f32", "f64"):
        assert lv.dot(dev([1, 2, 3], dt), dev([4, 5, 6], dt)) == 32
        assert lv.dot(lv.DenseVector.zeros(0, dt, device="cuda"), lv.DenseVector.zeros(0, dt, device="cuda")) == 0
        assert lv.norm2(dev([3, 4], dt)) == 5
        assert type(lv.norm2(dev([3, 4], dt))) is NP[dt]
        assert lv.sum(dev(range(1, 101), dt)) == 5050
        x = dev([1, 2, 3], dt)
        lv.scal(2, x)
        assert x.to_values() == [2, 4, 6]
    a, b, c = dev([1] * 5, "f32"), dev([5] * 5, "f32"), dev([1, 2, 3, 4, 5], "f32")
    d = lv.DenseVector.zeros(5, "f32", device="cuda")
    d.assign(a + (b - c))
    assert d.to_values() == [5, 4, 3, 2, 1]


def test_zero_length():
    x = lv.DenseVector.zeros(0, "f32", device="cuda")
    y = lv.DenseVector.zeros(0, "f32", device="cuda")
    lv.axpy(2.0, x, y)
    got = lv.dot(x, y)
    assert got == 0 and type(got) is np.float32


def test_aot_and_jit_kernels_agree_bit_for_bit():
    """Every compiled-in table entry equals the NVRTC build of its signature
    (proves each table type matches its signature string)."""
    g = np.random.default_rng(5)
    lib = _native.lib()
    n = 10_007
    for dt in ("f32", "f64"):
        ops = [g.uniform(-1, 1, n).astype(NP[dt]) for _ in range(4)]
        cases = [
            lambda v, d: d.assign(v[0]),
            lambda v, d: d.assign(1.5 * v[0]),
            lambda v, d: d.assign(v[0] + 0.75 * v[1]),
            lambda v, d: d.assign(0.75 * v[0] + v[1]),
            lambda v, d: d.assign(v[0] + v[1]),
            lambda v, d: d.assign(v[0] - v[1]),
            lambda v, d: d.assign(v[0] * v[1]),
            lambda v, d: d.assign(v[0] + (v[1] - v[2])),
            lambda v, d: d.assign(1.25 * v[0] + -0.5 * (v[1] - v[2])),
            lambda v, d: d.assign(1.25 * (v[0] + v[1]) - 0.5 * (v[2] - v[3]) + 0.3 * v[0]),
            lambda v, d: d.assign(1.25 * v[0] + -0.5 * v[1]),
            lambda v, d: d.assign(v[0] - 0.75 * v[1]),
        ]
        for k, case in enumerate(cases):
            outs = []
            for force in (0, 1):
                lib.salt_set_force_jit(force)
                try:
                    vecs = [dev(a, dt) for a in ops]
                    d = lv.DenseVector.zeros(n, dt, device="cuda")
                    case(vecs, d)
                    outs.append(d.to_array())
                finally:
                    lib.salt_set_force_jit(0)
            assert outs[0].tobytes() == outs[1].tobytes(), (dt, k)
        for force in (0, 1):
            lib.salt_set_force_jit(force)
            try:
                vecs = [dev(a, dt) for a in ops]
                x0, x1, x2 = (as_node(v) for v in vecs[:3])
                cg = AssignReduceNode(AssignNode(x1, x1 - ScaleNode(0.5, x0)), SumNode(x1 * x1))
                r = (lv.dot(vecs[0], vecs[1]), lv.sum(vecs[0]), lv.norm2(vecs[0]),
                     lv.axpy_dot(0.5, vecs[0], vecs[1], vecs[2]),
                     execute_reduce(SumNode((x0 - x1) * (x0 - x1))),
                     execute_reduce(SumNode(x0 * x1 * x2)),
                     lv.execute_assign_reduce(cg))
            finally:
                lib.salt_set_force_jit(0)
            if force == 0:
                r0 = r
            else:
                assert [x.tobytes() for x in r] == [x.tobytes() for x in r0], dt


def test_arbitrary_trees_through_jit():
    g = np.random.default_rng(6)
    n = 5000
    for dt in ("f32", "f64"):
        a, b, c, e = (g.uniform(-1, 1, n).astype(NP[dt]) for _ in range(4))
        A, B, C, E = (dev(v, dt) for v in (a, b, c, e))
        d = lv.DenseVector.zeros(n, dt, device="cuda")
        d.assign(((A - B) * (C + E)) * 0.5 - (A * A - 3.0 * (E - C)))
        want = restate.eval_sig("L0 L1 - L2 L3 + * S0 * L0 L0 * S1 L3 L2 - * - -",
                                [a, b, c, e], [0.5, 3.0], dt)
        assert same_bits(d.to_array(), want), dt
        r = execute_reduce(SumNode((as_node(A) - as_node(B)) * (as_node(C) + as_node(E))))
        exact = restate.exact_reduce("L0 L1 - L2 L3 + *", [a, b, c, e], [], dt)
        assert abs(float(r) - exact) <= TOL[dt] * abs(exact)


@pytest.mark.parametrize("dt", ["f32", "f64"])
def test_misaligned_views_and_ragged_lengths(dt):
    """Views starting at every element offset inside a 32-byte vector (the
    kernel's scalar head / V=1 fallback) and lengths around vector and
    block boundaries."""
    g = np.random.default_rng(7)
    base_n = 300_016
    a, b, c = (g.uniform(-1, 1, base_n).astype(NP[dt]) for _ in range(3))
    ta, tb, tc = (torch.from_numpy(v).cuda() for v in (a, b, c))
    td = torch.zeros(base_n, dtype=ta.dtype, device="cuda")
    vec = 32 // np.dtype(NP[dt]).itemsize
    for oa, ob, oc, od in [(0, 0, 0, 0), (1, 1, 1, 1), (vec - 1,) * 4, (1, 2, 3, 0), (0, 1, 0, 1)]:
        # 2,048 (f64) / 4,096 (f32) elements: one tile of the V = 1 kernels, which run
        # whole tiles only (the ragged end joins the scalar tail)
        # (up to 2^17 elements the small V = 1 assignment kernels run: 512-element tiles)
        for n in (0, 1, vec - 1, vec, vec + 1, 511, 512, 513, 2047, 2048, 2049, 4095, 4096, 4097, 8192, 65_537,
                  (1 << 17) + 5, 300_001):
            A = lv.DenseVector.from_tensor(ta[oa : oa + n])
            B = lv.DenseVector.from_tensor(tb[ob : ob + n])
            C = lv.DenseVector.from_tensor(tc[oc : oc + n])
            D = lv.DenseVector.from_tensor(td[od : od + n])
            D.assign(1.5 * A + -0.25 * (B - C))
            want = restate.eval_sig("S0 L0 * S1 L1 L2 - * +", [a[oa:oa + n], b[ob:ob + n], c[oc:oc + n]],
                                    [1.5, -0.25], dt)
            assert same_bits(D.to_array(), want), (oa, ob, oc, od, n)
            r = lv.dot(A, B)
            exact = restate.exact_sum((a[oa:oa + n] * b[ob:ob + n]))
            if exact != 0:
                assert abs(float(r) - exact) <= TOL[dt] * abs(exact), (oa, ob, n)


def test_exact_aliasing_inplace():
    g = np.random.default_rng(8)
    for dt in ("f32", "f64"):
        for n in (1, 100, 4099, 1 << 20):
            x = g.uniform(-1, 1, n).astype(NP[dt])
            y = g.uniform(-1, 1, n).astype(NP[dt])
            X, Y = dev(x, dt), dev(y, dt)
            lv.axpy(0.3, X, Y)
            assert same_bits(Y.to_array(), restate.eval_sig("L0 S0 L1 * +", [y, x], [0.3], dt))
            lv.scal(-1.75, X)
            assert same_bits(X.to_array(), restate.eval_sig("S0 L0 *", [x], [-1.75], dt))
            # identities the reference pins (test_ops.py:52-87)
            Y2 = dev(y, dt)
            lv.axpy(0, X, Y2)
            assert Y2.to_array().tobytes() == y.tobytes()
            X2 = dev(x, dt)
            lv.scal(1, X2)
            assert X2.to_array().tobytes() == x.tobytes()


def test_counting_vector_traffic_matches_reference():
    # reference test_acceptance.py:222-243 and test_engine.py:468-485
    x = lv.CountingVector.from_values(range(1000), device="cuda")
    out = lv.CountingVector.zeros(1000, device="cuda")
    lv.scaled_copy(1.25, x, out)
    assert (x.read_count, out.write_count, out.read_count) == (1000, 1000, 0)
    a, b, c = (lv.CountingVector.from_values(range(1000), device="cuda") for _ in range(3))
    d = lv.CountingVector.zeros(1000, device="cuda")
    d.assign(a + (b - c))
    assert a.read_count + b.read_count + c.read_count == 3000
    assert d.write_count == 1000 and d.read_count == 0
    a = lv.CountingVector.from_values(range(300), device="cuda")
    d = lv.CountingVector.zeros(300, device="cuda")
    d.assign(a + a)
    assert a.read_count == 600
    assert d.to_values() == [2.0 * i for i in range(300)]


def test_call_trace_golden_and_values():
    import json

    meta, z = golden("traces")
    for ci, (kind, n, dt, width, unroll, packages) in enumerate(meta):
        x = lv.DenseVector.from_values(np.arange(n), dt, device="cuda")
        y = lv.DenseVector.from_values(np.arange(n)[::-1].copy(), dt, device="cuda")
        if kind == "assign_scale":
            root = AssignNode(as_node(y), ScaleNode(2.0, as_node(x)))
        elif kind == "assign_axpy":
            root = AssignNode(as_node(y), as_node(y) + ScaleNode(0.5, as_node(x)))
        else:
            root = SumNode(as_node(x) * as_node(y))
        backend = lv.scalar_backend(dt) if width == 1 else lv.wide_backend(dt, width)
        opts = {"backend": backend}
        if unroll is not None:
            opts["unroll"] = unroll
        if packages is not None:
            opts["packages"] = packages
        tr = lv.call_trace(root, **opts)
        enc = [[e.kind, -1 if e.index is None else e.index, -1 if e.slot is None else e.slot] for e in tr]
        assert enc == json.loads(str(z[f"case{ci}"])), ci
        if kind == "assign_scale":
            assert y.to_values() == [2.0 * i for i in range(n)]


def test_host_vectors_stream_through_gpu():
    """Pinned-host vectors: chunked H2D -> fused kernel -> D2H (the
    end-to-end path) gives the same bits as the device path."""
    g = np.random.default_rng(9)
    for dt in ("f32", "f64"):
        for n in (0, 5, 1 << 20, (1 << 23) + 77, 3 * (1 << 23) + 5):
            a, b, c = (g.uniform(-1, 1, n).astype(NP[dt]) for _ in range(3))
            H = [lv.DenseVector.from_values(v, dt, device="cpu") for v in (a, b, c)]
            assert H[0].tensor.is_pinned() or n == 0
            out = lv.DenseVector.zeros(n, dt, device="cpu")
            out.assign(0.5 * H[0] + 2.0 * (H[1] - H[2]))
            want = restate.eval_sig("S0 L0 * S1 L1 L2 - * +", [a, b, c], [0.5, 2.0], dt)
            assert same_bits(out.to_array(), want), (dt, n)
            r = lv.dot(H[0], H[1])
            exact = restate.exact_sum(a * b)
            if exact != 0:
                assert abs(float(r) - exact) <= TOL[dt] * abs(exact), (dt, n)
            # in-place on host (dest aliases a leaf)
            lv.axpy(0.25, H[0], H[1])
            assert same_bits(H[1].to_array(), restate.eval_sig("L0 S0 L1 * +", [b, a], [0.25], dt))


def test_lazy_reduction_returns_device_scalar():
    x = dev(np.arange(1, 101), "f64")
    r = lv.dot(x, x, lazy=True)
    assert isinstance(r, lv.DeviceScalar)
    assert r.item() == sum(i * i for i in range(1, 101))
    r32 = lv.sum(dev(np.arange(1, 101), "f32"), lazy=True)
    assert r32.item() == 5050 and type(r32.item()) is np.float32


def test_launches_are_counted_and_native():
    lib = _native.lib()
    before = lib.salt_launch_count()
    x = dev(np.ones(1000), "f32")
    lv.scal(2.0, x)
    lv.dot(x, x)
    torch.cuda.synchronize()
    assert lib.salt_launch_count() - before == 2


def test_cuda_graph_capture_of_fused_steps():
    """Launch-bound loops (small n) can be captured in a CUDA graph: the
    kernels go to the caller's current stream, lazy reductions never
    synchronise, and the reduction workspace resets itself in-kernel."""
    n = 1 << 16
    g = np.random.default_rng(10)
    x, y, z = (g.standard_normal(n) for _ in range(3))
    X, Y, Z = dev(x, "f64"), dev(y, "f64"), dev(z, "f64")
    eager = []
    for _ in range(5):
        eager.append(float(lv.axpy_dot(0.25, X, Y, Z)))
    y_eager = Y.to_array()
    Y2 = dev(y, "f64")
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        lv.axpy_dot(0.25, X, Y2, Z, lazy=True)  # warm-up: JIT/occupancy/workspace
    torch.cuda.current_stream().wait_stream(s)
    Y2.tensor.copy_(torch.from_numpy(y))
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        outs = [lv.axpy_dot(0.25, X, Y2, Z, lazy=True) for _ in range(5)]
    graph.replay()
    torch.cuda.synchronize()
    assert [float(o.item()) for o in outs] == eager
    assert Y2.to_array().tobytes() == y_eager.tobytes()


def test_graphs_with_reductions_replay_concurrently():
    """Each captured graph gets its own reduction workspace:
    two graphs whose reductions combine through tickets (multi-CTA n),
    replayed at the same time on two streams, plus eager reductions on the
    default stream meanwhile, all give the eager bits."""
    from paper_1109_1264_b200 import runtime

    n = (1 << 23) + 5
    g = np.random.default_rng(12)
    xs = [dev(g.standard_normal(n), "f64") for _ in range(4)]
    want = [float(lv.dot(xs[0], xs[1])), float(lv.dot(xs[2], xs[3])), float(lv.norm2(xs[0]))]
    graphs, outs = [], []
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        lv.dot(xs[0], xs[1], lazy=True)  # warm-up outside capture
    torch.cuda.current_stream().wait_stream(side)
    before = len(runtime._capture_workspaces)
    for a, b in ((0, 1), (2, 3)):
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr):
            outs.append(lv.dot(xs[a], xs[b], lazy=True))
        graphs.append(gr)
    assert len(runtime._capture_workspaces) == before + 2
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    for _ in range(20):
        for gr, st in zip(graphs, streams):
            st.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(st):
                gr.replay()
        assert float(lv.norm2(xs[0])) == want[2]  # eager, default stream, meanwhile
        for st in streams:
            torch.cuda.current_stream().wait_stream(st)
        torch.cuda.synchronize()
        assert [float(o.item()) for o in outs] == want[:2]


def test_special_reductions_match_reference():
    """inf / -inf / NaN / overflow in reductions: the compensated sum falls
    back to the plain IEEE sum, giving the reference's inf / NaN results."""
    meta, z = golden("special_reductions")
    for cname, dt, n in meta:
        key = f"{cname}|{dt}"
        X = dev(z[f"{key}|x"], dt)
        assert same_bits(np.array([lv.sum(X)]), z[f"{key}|sum"]), key
        assert same_bits(np.array([lv.dot(X, X)]), z[f"{key}|dot"]), key


def test_concurrent_evaluation_from_threads():
    """One expression value evaluated concurrently from several threads, each
    on its own CUDA stream (reference contract: expressions.py:17-21).  The
    C ABI is re-entrant and reduction workspaces are per stream."""
    import threading

    n = 1 << 20
    g = np.random.default_rng(11)
    a, b = g.uniform(-1, 1, n), g.uniform(-1, 1, n)
    A, B = dev(a, "f64"), dev(b, "f64")
    expr = 1.5 * A - 0.5 * (B - A)
    want = restate.eval_sig("S0 L0 * S1 L1 L0 - * -", [a, b], [1.5, 0.5], "f64")
    exact = restate.exact_sum(a * b)
    errors = []

    def worker(k):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                d = lv.DenseVector.empty(n, "f64", device="cuda")
                for _ in range(20):
                    d.assign(expr)
                    r = lv.dot(A, B)
                    assert abs(float(r) - exact) <= 1e-12 * abs(exact)
                s.synchronize()
                assert d.to_array().tobytes() == want.tobytes()
        except Exception as exc:  # collected for the main thread
            errors.append((k, repr(exc)))

    ts = [threading.Thread(target=worker, args=(k,)) for k in range(6)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errors, errors


def test_fused_axpy_dot_on_host_vectors():
    g = np.random.default_rng(12)
    for dt in ("f32", "f64"):
        n = (1 << 23) * 2 + 99
        x, y, z = (g.standard_normal(n).astype(NP[dt]) for _ in range(3))
        X, Y, Z = (lv.DenseVector.from_values(v, dt, device="cpu") for v in (x, y, z))
        r = lv.axpy_dot(-0.375, X, Y, Z)
        y_new = restate.eval_sig("L0 S0 L1 * +", [y, x], [-0.375], dt)
        assert same_bits(Y.to_array(), y_new)
        exact = restate.exact_sum((y_new * z))
        assert abs(float(r) - exact) <= TOL[dt] * abs(exact)


def test_no_writes_outside_the_destination():
    """compute-sanitizer is closed on this pool, so out-of-bounds writes are
    checked with canaries: destinations are views inside a larger buffer
    filled with a sentinel; after every kind of evaluation (vector body,
    scalar head/tail, V=1 fallback, fused assign+reduce) everything outside
    the view still holds the sentinel."""
    g = np.random.default_rng(13)
    for dt in ("f32", "f64"):
        tdt = torch.float32 if dt == "f32" else torch.float64
        for n in (1, 3, 8, 9, 31, 1023, 1025, 65_541):
            for off in (0, 1, 2, 5):
                src = [torch.from_numpy(g.uniform(-1, 1, n + 64)).to(tdt).cuda() for _ in range(3)]
                buf = torch.full((n + 64,), 12345.0, dtype=tdt, device="cuda")
                a, b, c = (lv.DenseVector.from_tensor(t[off:off + n]) for t in src)
                mis = (off + 1) % 4  # also a misalignment different from the sources
                for doff in (off, mis):
                    buf.fill_(12345.0)
                    d = lv.DenseVector.from_tensor(buf[doff:doff + n])
                    d.assign(0.5 * a - b * c)
                    lv.axpy_dot(0.5, a, d, b)
                    outside = torch.cat([buf[:doff], buf[doff + n:]])
                    assert bool((outside == 12345.0).all()), (dt, n, off, doff)
                    assert bool((buf[doff:doff + n] != 12345.0).all())


def test_c_fast_path_matches_python_path():
    """The C host fast path (csrc/fastpath.c) is active for device vectors
    and produces exactly what the Python lowering path produces (plan
    keywords force the Python path)."""
    fast = _native.fastpath()
    assert fast is not None
    g = np.random.default_rng(14)
    for dt in ("f32", "f64"):
        n = 100_003
        a, b, c = (dev(g.uniform(-1, 1, n), dt) for _ in range(3))
        d1, d2 = (lv.DenseVector.zeros(n, dt, device="cuda") for _ in range(2))
        assert fast.assign(d1, (1.5 * a - b * c).left) is True  # a bare ScaleNode tree
        d1.assign(1.5 * a - b * c)
        d2.assign(1.5 * a - b * c, unroll=1)
        assert d1.to_array().tobytes() == d2.to_array().tobytes()
        r1, r2 = lv.dot(a, b), lv.dot(a, b, unroll=1)
        assert r1.tobytes() == r2.tobytes() and type(r1) is type(r2) is NP[dt]
        assert lv.norm2(a).tobytes() == lv.norm2(a, unroll=1).tobytes()
        lz = lv.dot(a, b, lazy=True)
        assert isinstance(lz, lv.DeviceScalar) and lz.item().tobytes() == r1.tobytes()
        y1, y2 = dev(b.to_array(), dt), dev(b.to_array(), dt)
        s1, s2 = lv.axpy_dot(0.5, a, y1, c), lv.axpy_dot(0.5, a, y2, c, unroll=1)
        assert s1.tobytes() == s2.tobytes()
        assert y1.to_array().tobytes() == y2.to_array().tobytes()
