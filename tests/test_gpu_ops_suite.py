"""The reference's unit-test surface for the named operations and the
engine's result semantics, restated against the B200 path.

Test names follow the reference's tests (pkg/tests/test_ops.py,
test_engine.py, test_vectors.py) so a reader can line them up; the cases,
values and seeds are this repository's own, and the expected results come
from oracle/ (test infrastructure) or exact small-integer arithmetic.
Everything below runs the CUDA kernels (vectors resident on cuda:0)."""

import numpy as np
import pytest

import paper_1109_1264_b200 as lv
from oracle import restate
from paper_1109_1264_b200 import LengthMismatchError, _native
from paper_1109_1264_b200.engine import execute_assign, execute_reduce
from paper_1109_1264_b200.expressions import AssignNode, Leaf, SumNode, as_node
from paper_1109_1264_b200.lanes import scalar_backend, wide_backend

pytestmark = pytest.mark.gpu
DTYPES = ("f32", "f64")
NPT = {"f32": np.float32, "f64": np.float64}


def vec(values, dtype="f32"):
    return lv.DenseVector.from_values(values, dtype, device="cuda")


# ------------------------------------------------------------ ops.py surface
@pytest.mark.parametrize("dtype", DTYPES)
def test_dot(dtype):
    assert lv.dot(vec([2, -1, 4, 3], dtype), vec([1, 5, 2, -2], dtype)) == -1  # 2-5+8-6
    assert lv.dot(vec([7, 8], dtype), vec([3, 1], dtype)) == 29
    assert lv.dot(lv.DenseVector.zeros(0, dtype, device="cuda"),
                  lv.DenseVector.zeros(0, dtype, device="cuda")) == 0


def test_dot_length_mismatch():
    with pytest.raises(LengthMismatchError):
        lv.dot(vec([1, 2, 3, 4]), vec([1, 2, 3]))


@pytest.mark.parametrize("dtype", DTYPES)
def test_dot_returns_element_typed_scalar(dtype):
    r = lv.dot(vec([3], dtype), vec([5], dtype))
    assert type(r) is NPT[dtype] and r == 15


@pytest.mark.parametrize("dtype", DTYPES)
def test_dot_large_matches_compensated_reference(dtype):
    g = np.random.default_rng(8191)
    n = 1_000_003
    xs, ys = (g.uniform(0.1, 1.1, n).astype(NPT[dtype]) for _ in range(2))
    got = float(lv.dot(vec(xs, dtype), vec(ys, dtype)))
    want = restate.exact_sum(restate.eval_sig("L0 L1 *", [xs, ys], [], dtype))
    assert abs(got - want) <= {"f32": 1e-5, "f64": 1e-12}[dtype] * abs(want)


@pytest.mark.parametrize("dtype", DTYPES)
def test_scal(dtype):
    x = vec([1.5, -2, 4], dtype)
    lv.scal(-2, x)
    assert x.to_values() == [-3, 4, -8]
    lv.scal(0, x)
    assert x.to_array().tolist() == [0, -0.0, 0]


def test_scal_by_one_is_bit_exact_identity():
    g = np.random.default_rng(5)
    for dtype in DTYPES:
        values = g.standard_normal(70_001).astype(NPT[dtype])
        x = vec(values, dtype)
        lv.scal(1, x)
        assert x.to_array().tobytes() == values.tobytes()


@pytest.mark.parametrize("dtype", DTYPES)
def test_axpy(dtype):
    x, y = vec([1, -2, 3], dtype), vec([10, 10, 10], dtype)
    lv.axpy(-3, x, y)
    assert y.to_values() == [7, 16, 1]
    with pytest.raises(LengthMismatchError):
        lv.axpy(1, vec([1, 2], dtype), vec([1, 2, 3], dtype))


def test_axpy_alpha_zero_leaves_y_bit_exact():
    g = np.random.default_rng(6)
    for dtype in DTYPES:
        x = vec(g.standard_normal(12_345).astype(NPT[dtype]), dtype)
        yv = g.standard_normal(12_345).astype(NPT[dtype])
        y = vec(yv, dtype)
        lv.axpy(0, x, y)
        assert y.to_array().tobytes() == yv.tobytes()


def test_axpy_matches_scalar_loop_bit_exactly():
    g = np.random.default_rng(7)
    for dtype in DTYPES:
        xv, yv = (g.uniform(-1, 1, 257).astype(NPT[dtype]) for _ in range(2))
        x, y = vec(xv, dtype), vec(yv, dtype)
        want = restate.oracle_axpy(NPT[dtype](0.7), list(xv), list(yv))
        lv.axpy(0.7, x, y)
        assert y.to_array().tobytes() == np.array(want, dtype=NPT[dtype]).tobytes()


@pytest.mark.parametrize("dtype", DTYPES)
def test_scaled_copy(dtype):
    x = vec([2, -4, 8], dtype)
    out = lv.DenseVector.zeros(3, dtype, device="cuda")
    lv.scaled_copy(0.5, x, out)
    assert out.to_values() == [1, -2, 4]
    assert x.to_values() == [2, -4, 8]
    with pytest.raises(LengthMismatchError):
        lv.scaled_copy(1, vec([1], dtype), lv.DenseVector.zeros(3, dtype, device="cuda"))


def test_scaled_copy_by_one_is_bit_exact_copy():
    g = np.random.default_rng(8)
    for dtype in DTYPES:
        values = g.standard_normal(3001).astype(NPT[dtype])
        x, out = vec(values, dtype), lv.DenseVector.zeros(3001, dtype, device="cuda")
        lv.scaled_copy(1, x, out)
        assert out.to_array().tobytes() == values.tobytes()


@pytest.mark.parametrize("dtype", DTYPES)
def test_norm2(dtype):
    assert lv.norm2(vec([5, 12], dtype)) == 13
    assert lv.norm2(vec([1, 2, 2], dtype)) == 3
    assert lv.norm2(lv.DenseVector.zeros(77, dtype, device="cuda")) == 0
    assert type(lv.norm2(vec([6, 8], dtype))) is NPT[dtype]


@pytest.mark.parametrize("dtype", DTYPES)
def test_sum(dtype):
    assert lv.sum(lv.DenseVector.zeros(33, dtype, device="cuda")) == 0
    assert lv.sum(vec(range(-10, 201), dtype)) == sum(range(-10, 201))


def test_options_pass_through_to_the_engine():
    x, y = vec([3, 1, 4, 1, 5, 9, 2]), vec([2, 7, 1, 8, 2, 8, 1])
    base = lv.dot(x, y)
    for opts in (dict(unroll=4), dict(backend=scalar_backend("f32")),
                 dict(backend=wide_backend("f32", 4), unroll=2, packages=2), dict(stepped=True)):
        assert lv.dot(x, y, **opts) == base


def test_inplace_ops_accept_overrides():
    x = vec(range(50), "f64")
    lv.scal(3, x, unroll=2, stepped=True)
    assert x.to_values() == [3.0 * i for i in range(50)]
    y = vec([1.0] * 50, "f64")
    lv.axpy(2, x, y, unroll=8)
    assert y.to_values() == [1.0 + 6.0 * i for i in range(50)]


# ------------------------------------------------ engine.py result semantics
def test_add_of_difference_example():
    a, b, c = vec([10, 20, 30, 40]), vec([1, 2, 3, 4]), vec([4, 3, 2, 1])
    d = lv.DenseVector.zeros(4, "f32", device="cuda")
    execute_assign(AssignNode(Leaf(d), as_node(a) + (as_node(b) - as_node(c))))
    assert d.to_values() == [7, 19, 31, 43]


@pytest.mark.parametrize("dtype", DTYPES)
def test_zero_length_assign_and_reduce(dtype):
    e = lv.DenseVector.zeros(0, dtype, device="cuda")
    e.assign(2.0 * e + e)  # no-op
    r = execute_reduce(SumNode(as_node(e) * as_node(e)))
    assert r == 0 and type(r) is NPT[dtype]


def test_dot_small_values():
    assert lv.dot(vec([0.5, 0.25], "f64"), vec([4, 8], "f64")) == 4


def test_masked_main_loop_plus_remainder_covers_everything():
    # every length around the vector width / tile boundaries is evaluated in full
    for dtype in DTYPES:
        for n in (1, 3, 7, 8, 9, 15, 16, 17, 31, 33, 255, 257, 2047, 2049, 8191, 8193):
            x = vec(np.arange(n), dtype)
            y = lv.DenseVector.zeros(n, dtype, device="cuda")
            y.assign(1.0 * x + x)
            assert y.to_values() == [2.0 * i for i in range(n)], (dtype, n)
            assert lv.sum(x) == n * (n - 1) // 2


def test_packages_do_not_change_results():
    g = np.random.default_rng(9)
    a, b = (vec(g.uniform(-1, 1, 999).astype(np.float32)) for _ in range(2))
    base = lv.DenseVector.zeros(999, "f32", device="cuda")
    base.assign(a * b - a)
    for packages in (1, 2, 4):
        d = lv.DenseVector.zeros(999, "f32", device="cuda")
        d.assign(a * b - a, unroll=4, packages=packages)
        assert d.to_array().tobytes() == base.to_array().tobytes()


def test_exact_aliasing_source_equals_destination():
    g = np.random.default_rng(10)
    for dtype in DTYPES:
        xv, yv = (g.uniform(-1, 1, 4097).astype(NPT[dtype]) for _ in range(2))
        x, y = vec(xv, dtype), vec(yv, dtype)
        y.assign(y * x + y)  # destination read as a leaf, written once
        want = restate.eval_sig("L0 L1 * L0 +", [yv, xv], [], dtype)
        assert y.to_array().tobytes() == want.tobytes()


def test_each_leaf_occurrence_is_read_exactly_once():
    # a vector used several times is loaded once per element by the fused kernel
    x = vec(np.arange(1, 1025), "f64")
    y = lv.DenseVector.zeros(1024, "f64", device="cuda")
    before = _native.lib().salt_launch_count()
    y.assign(x * x + x - 3.0 * x)
    assert _native.lib().salt_launch_count() - before == 1
    i = np.arange(1, 1025, dtype=np.float64)
    assert y.to_array().tobytes() == (i * i + i - 3.0 * i).tobytes()
    t = lv.traffic(AssignNode(Leaf(y), x * x + x - 3.0 * x))
    assert t["vectors_read"] == 1 and t["vectors_written"] == 1 and t["bytes"] == 2 * 8 * 1024


def test_reduction_matches_oracle_within_tolerance():
    g = np.random.default_rng(11)
    for dtype in DTYPES:
        for n in (5, 1000, 100_001, 2_000_003):
            xs = g.standard_normal(n).astype(NPT[dtype])
            got = float(lv.sum(vec(xs, dtype)))
            want = restate.exact_sum(xs)
            scale = restate.exact_sum(np.abs(xs))
            assert abs(got - want) <= {"f32": 1e-5, "f64": 1e-12}[dtype] * max(abs(want), 1e-3 * scale)


# ------------------------------------------------------ vectors.py surface
def test_assign_evaluates_expressions():
    a, b = vec([1, 2, 3], "f64"), vec([4, 5, 6], "f64")
    d = lv.DenseVector.zeros(3, "f64", device="cuda")
    d.assign(-(a - b) * 2.0)
    assert d.to_values() == [6, 6, 6]


def test_assign_accepts_plan_overrides():
    a = vec([1, 2, 3, 4, 5])
    d = lv.DenseVector.zeros(5, "f32", device="cuda")
    d.assign(a + a, unroll=2, packages=1, backend=wide_backend("f32", 8))
    assert d.to_values() == [2, 4, 6, 8, 10]


def test_named_ops_fast_path_is_taken_and_matches_the_node_path(monkeypatch):
    """ops.* on plain device vectors go straight to the C fast path (no
    node objects, csrc/fastpath.c `op`) and give the node path's bits; the
    alpha coercion matches ScaleNode's for every scalar type."""
    import paper_1109_1264_b200.ops as ops_mod

    g = np.random.default_rng(12)
    alphas = [0.7, 3, True, np.float32(-1.3), np.float64(2.0 ** -30 + 1.0), 1e300]
    for dtype in DTYPES:
        xv, yv = (g.standard_normal(50_003).astype(NPT[dtype]) for _ in range(2))

        def run():
            out = []
            for a in alphas:
                x, y, o = vec(xv, dtype), vec(yv, dtype), lv.DenseVector.zeros(50_003, dtype, device="cuda")
                lv.axpy(a, x, y)
                lv.scal(a, x)
                lv.scaled_copy(a, y, o)
                out += [x.to_array(), y.to_array(), o.to_array()]
            x, y = vec(xv, dtype), vec(yv, dtype)
            out += [np.array([lv.dot(x, y), lv.dot(x, x), lv.sum(x), lv.norm2(y),
                              lv.dot(x, y, lazy=True).item(), lv.norm2(x, lazy=True).item()])]
            return out

        calls = []
        real_assign, real_reduce = ops_mod.execute_assign, ops_mod.execute_reduce
        monkeypatch.setattr(ops_mod, "execute_assign", lambda *a, **k: calls.append(1) or real_assign(*a, **k))
        monkeypatch.setattr(ops_mod, "execute_reduce", lambda *a, **k: calls.append(1) or real_reduce(*a, **k))
        fast = run()
        assert not calls  # every call above took the C fast path
        monkeypatch.setattr(_native, "_fast", None)
        slow = run()
        assert calls
        monkeypatch.undo()
        for u, v in zip(fast, slow):
            assert u.tobytes() == v.tobytes()
