"""Host-side API parity with the reference (CPU, no GPU needed).

Mirrors the reference's unit tests for lanes, vectors, expressions, plans
and traces (pkg/tests/test_{lanes,vectors,expressions,engine}.py): the same
names, argument meanings, validation and exceptions — everything that is
decided before a kernel is launched.  Vectors here live in host memory
(device="cpu"); evaluating a tree over them needs a GPU and is covered by
the gpu-marked tests.
"""

import json

import numpy as np
import pytest

import paper_1109_1264_b200 as lv
from conftest import golden
from paper_1109_1264_b200.engine import (
    DEFAULT_REGISTER_BUDGET,
    PlanError,
    UnrollPlan,
    _trace_events,
    execute_assign,
    execute_reduce,
    masked_length,
    select_plan,
)
from paper_1109_1264_b200.expressions import (
    AddNode,
    AssignNode,
    AssignReduceNode,
    Leaf,
    LengthMismatchError,
    MulNode,
    ScaleNode,
    SubNode,
    SumNode,
    as_node,
    combine_partials,
    common_length,
    lower,
)
from paper_1109_1264_b200.lanes import (
    CONTAINER_ALIGNMENT,
    DEVICE_ALIGNMENT,
    as_dtype,
    dtype_name,
    horizontal_sum,
    scalar_backend,
    wide_backend,
)


def hv(values, dtype="f32"):
    return lv.DenseVector.from_values(values, dtype, device="cpu")


# ---------------------------------------------------------------- lanes
def test_dtype_spellings_and_rejections():
    assert as_dtype("f32") == np.float32 and as_dtype(np.float64) == np.float64
    for bad in ("f16", np.int32, "int64", complex):
        with pytest.raises(TypeError):
            as_dtype(bad)
    for name in ("f32", "f64"):
        assert dtype_name(as_dtype(name)) == name


def test_backend_validation_and_defaults():
    assert wide_backend("f32").width == 16 and wide_backend("f64").width == 8
    assert scalar_backend("f32").caps.width == 1
    with pytest.raises(ValueError):
        lv.LaneBackend("f32", 3, True)
    with pytest.raises(ValueError):
        lv.LaneBackend("f64", 16, True)  # 128 B > 64 B block
    with pytest.raises(ValueError):
        lv.LaneBackend("f32", 4, False)
    with pytest.raises(ValueError):
        wide_backend("f32", 1)
    be = wide_backend("f32", 4)
    assert type(be.scalar(0.1)) is np.float32
    with pytest.raises(TypeError):
        be.scalar("3")
    assert horizontal_sum(be.splat(1)) == 4


def test_horizontal_sum_is_left_to_right():
    lanes = np.array([1e8, 1.0, -1e8, 1.0], dtype=np.float32)
    expected = ((np.float32(1e8) + np.float32(1.0)) + np.float32(-1e8)) + np.float32(1.0)
    assert horizontal_sum(lv.LaneVector(lanes)) == expected


# ---------------------------------------------------------------- vectors
@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_vectors_basics(dtype):
    v = lv.DenseVector.zeros(7, dtype, device="cpu")
    assert len(v) == 7 and v.to_values() == [0] * 7
    assert v.dtype == as_dtype(dtype)
    w = hv([1.5, -2.0, 3.25], dtype)
    assert w.to_values() == [1.5, -2.0, 3.25]
    assert all(type(x) is as_dtype(dtype).type for x in w.to_values())
    assert lv.DenseVector.zeros(0, dtype, device="cpu").to_values() == []
    with pytest.raises(ValueError):
        lv.DenseVector.zeros(-1, device="cpu")


@pytest.mark.parametrize("n", [1, 2, 3, 17, 64, 129, 1000])
def test_storage_alignment(n):
    v = lv.DenseVector.zeros(n, "f64", device="cpu")
    assert v.address % DEVICE_ALIGNMENT == 0
    assert v.address % CONTAINER_ALIGNMENT == 0


def test_element_access_and_errors():
    v = hv([1, 2, 3])
    assert v.get(1) == 2
    v.set(1, 9)
    assert v[1] == 9
    v[2] = 7.5
    assert v.get(2) == 7.5
    for bad in (-1, 3, 100):
        with pytest.raises(IndexError):
            v.get(bad)
        with pytest.raises(IndexError):
            v.set(bad, 0)
    z = lv.DenseVector.zeros(1, "f32", device="cpu")
    z.set(0, 0.1)
    assert type(z.get(0)) is np.float32 and z.get(0) == np.float32(0.1)
    arr = v.to_array()
    arr[0] = 99
    assert v.get(0) == 1
    b = lv.DenseVector.zeros(8, "f64", device="cpu")
    b.write_block(2, 6, np.array([1.0, 2.0, 3.0, 4.0]))
    assert list(b.read_block(2, 6)) == [1, 2, 3, 4]
    b.write_element(0, 5)
    assert b.read_element(3) == 2 and b.to_values() == [5, 0, 1, 2, 3, 4, 0, 0]


def test_operator_sugar_builds_nodes():
    x, y = hv([1, 2]), hv([3, 4])
    assert isinstance(x + y, AddNode)
    assert isinstance(x - y, SubNode)
    assert isinstance(x * y, MulNode)
    assert isinstance(2.5 * x, ScaleNode) and isinstance(x * 2.5, ScaleNode)
    assert isinstance(-x, ScaleNode)
    assert isinstance(np.float32(2.0) * x, ScaleNode)
    assert isinstance((x + y) - x * 2.0, SubNode)
    e = x + (y - x)
    assert isinstance(e.left, Leaf) and isinstance(e.right, SubNode)
    with pytest.raises(TypeError):
        _ = 1.0 + (x + x)
    with pytest.raises(TypeError):
        _ = (x + x) - 1.0
    with pytest.raises(TypeError):
        as_node([1, 2, 3])


def test_dtype_rules():
    x32, y64 = hv([1, 2]), hv([1, 2], "f64")
    with pytest.raises(TypeError):
        _ = x32 + y64
    with pytest.raises(TypeError):
        AssignNode(as_node(y64), as_node(x32))
    with pytest.raises(TypeError):
        AssignNode(as_node(x32) + as_node(x32), as_node(x32))
    node = ScaleNode(0.1, as_node(hv([1])))
    assert type(node.alpha) is np.float32 and node.alpha == np.float32(0.1)
    assert type(ScaleNode(np.float32(2.0), as_node(y64)).alpha) is np.float64


def test_register_footprints_match_reference():
    a, b, c = hv([1]), hv([2]), hv([3])
    assert as_node(a).register_footprint == 1
    assert (a + b).register_footprint == 2
    assert (2.0 * a).register_footprint == 2
    assert (a + (b - c)).register_footprint == 3
    assert SumNode(as_node(a) * as_node(b)).register_footprint == 3
    src = as_node(b) + 2.0 * as_node(a)
    assert AssignNode(as_node(c), src).register_footprint == 4


def test_common_length_checks_destination_too():
    a, b, short = hv([1, 2, 3]), hv([4, 5, 6]), hv([1, 2])
    assert common_length(a + b) == 3
    with pytest.raises(LengthMismatchError):
        common_length(a + short)
    with pytest.raises(LengthMismatchError):
        common_length(AssignNode(as_node(short), as_node(a) + as_node(b)))


def test_combine_partials_order():
    rows = [np.ones(4, dtype=np.float32), np.full(4, 2, dtype=np.float32)]
    assert combine_partials(rows, np.float32(3)) == 15
    assert combine_partials([], np.float32(1.5)) == np.float32(1.5)


# ---------------------------------------------------------------- lowering
def test_lowering_signatures_of_named_ops_and_configs():
    a, b, c, d = hv([1.0]), hv([2.0]), hv([3.0]), hv([4.0])
    assert lower(a + (b - c)).tokens == "L0 L1 L2 - +".split()
    lw = lower(1.5 * a + -0.5 * (b - c))
    assert lw.tokens == "S0 L0 * S1 L1 L2 - * +".split()
    assert lw.scalars == [1.5, -0.5]
    lw = lower(2.0 * (a + b) - 3.0 * (c - d) + 0.5 * a)
    assert " ".join(lw.tokens) == "S0 L0 L1 + * S1 L2 L3 - * - S2 L0 * +"
    assert lw.vectors == [a, b, c, d] and lw.occurrences == [2, 1, 1, 1]
    # axpy builds y + alpha*x (ops.py:32-36): y is leaf 0
    lw = lower(as_node(b) + ScaleNode(0.25, as_node(a)))
    assert " ".join(lw.tokens) == "L0 S0 L1 * +" and lw.vectors == [b, a]
    # scalars are coerced to the element type before lowering
    lw = lower(0.1 * a)
    assert lw.scalars == [float(np.float32(0.1))]
    # fused root: the destination inside the reduce tree reads D
    y, x, z = hv([1.0]), hv([2.0]), hv([3.0])
    lwa = lower(as_node(y) + ScaleNode(0.5, as_node(x)))
    lwr = lower(as_node(y) * as_node(z), parent=lwa, dest=y)
    assert " ".join(lwa.tokens) == "L0 S0 L1 * +" and " ".join(lwr.tokens) == "D0 L2 *"
    # multi-statement fusion: later statements read earlier destinations as D<k>
    p, q = hv([4.0]), hv([5.0])
    fz = lv.FusedNode([AssignNode(as_node(x), as_node(x) + 0.5 * as_node(p)),
                       AssignNode(as_node(y), as_node(y) - 0.5 * as_node(q) + as_node(x))],
                      SumNode(as_node(y) * as_node(y)))
    asig, rsig, lw2, dests = fz.lower()
    assert asig == "L0 S0 L1 * + ; L2 S1 L3 * - D0 +" and rsig == "D1 D1 *"
    assert lw2.vectors == [x, p, y, q] and dests == [x, y]


def test_building_touches_no_elements():
    a, b, c = (lv.CountingVector.from_values(range(64), device="cpu") for _ in range(3))
    expr = ((a + b) - c) * 2.0 + (b - a)
    assert expr.register_footprint > 0
    _ = lower(expr)
    assert all(v.read_count == 0 and v.write_count == 0 for v in (a, b, c))


# ---------------------------------------------------------------- plans
def test_masked_length_examples():
    assert masked_length(10, 2, 4) == 8
    assert masked_length(16, 2, 4) == 16
    assert masked_length(0, 8, 4) == 0
    assert masked_length(129, 8, 4) == 128
    assert masked_length(31, 1, 1) == 31


def test_select_plan_rules():
    caps = wide_backend("f32", 4).caps
    assert [select_plan(f, 100, caps).unroll for f in (2, 3, 4, 5, 16, 17)] == [8, 4, 4, 2, 1, 1]
    assert select_plan(2, 100, caps, register_budget=8).unroll == 4
    p = select_plan(4, 77, scalar_backend("f32").caps)
    assert (p.unroll, p.width, p.masked_length) == (1, 1, 77)
    p = select_plan(8, 100, caps, unroll=8, packages=4)
    assert (p.unroll, p.packages, p.masked_length) == (8, 4, 96)
    p = select_plan(4, 100, scalar_backend("f32").caps, unroll=8)
    assert (p.unroll, p.width) == (8, 1)
    for kw in ({"unroll": 3}, {"unroll": 16}, {"unroll": 4, "packages": 3},
               {"unroll": 2, "packages": 4}):
        with pytest.raises(PlanError):
            select_plan(2, 10, caps, **kw)
    with pytest.raises(PlanError):
        select_plan(0, 10, caps)
    with pytest.raises(PlanError):
        select_plan(2, -1, caps)
    assert DEFAULT_REGISTER_BUDGET == 16


def test_unroll_plan_invariants():
    p = UnrollPlan(4, 4, 2, 32)
    assert p.block == 16 and p.slots_per_package == 2
    for bad in ((3, 4, 1, 0), (4, 3, 1, 0), (4, 4, 3, 0), (4, 4, 1, 8), (4, 4, 1, -16)):
        with pytest.raises(PlanError):
            UnrollPlan(*bad)


def test_validation_raises_before_any_launch():
    """Every reference error is raised on the host, before libsalt is
    called — these run without a GPU."""
    x, y = hv(np.arange(20.0)), hv(np.arange(20.0))
    root = AssignNode(as_node(y), as_node(y) + ScaleNode(1.5, as_node(x)))
    with pytest.raises(PlanError):
        execute_assign(root, UnrollPlan(2, 4, 1, 16), backend=wide_backend("f32", 8))
    with pytest.raises(PlanError):
        execute_assign(root, UnrollPlan(2, 4, 1, 8), backend=wide_backend("f32", 4))
    with pytest.raises(PlanError):
        execute_assign(root, UnrollPlan(2, 4, 1, 16), backend=wide_backend("f32", 4), unroll=2)
    with pytest.raises(PlanError):
        execute_assign(root, backend=wide_backend("f64", 4))
    with pytest.raises(TypeError):
        execute_assign(root, backend="wide")
    with pytest.raises(TypeError):
        execute_assign(SumNode(as_node(x) * as_node(y)))
    with pytest.raises(TypeError):
        execute_reduce(root)
    with pytest.raises(LengthMismatchError):
        lv.dot(hv([1, 2]), hv([1, 2, 3]))
    with pytest.raises(LengthMismatchError):
        lv.axpy(1, hv([1]), hv([1, 2]))
    with pytest.raises(LengthMismatchError):
        lv.scaled_copy(1, hv([1]), lv.DenseVector.zeros(2, device="cpu"))
    with pytest.raises(TypeError):
        AssignReduceNode(SumNode(as_node(x)), SumNode(as_node(x)))


def test_trace_synthesis_matches_reference_golden():
    meta, z = golden("traces")
    for ci, (kind, n, dt, width, unroll, packages) in enumerate(meta):
        caps = (scalar_backend(dt) if width == 1 else wide_backend(dt, width)).caps
        if kind == "assign_scale":
            fp = 3
        elif kind == "assign_axpy":
            fp = 4
        else:
            fp = 3
        plan = select_plan(fp, n, caps, unroll=unroll, packages=packages)
        tr = _trace_events(plan, n, kind.startswith("reduce"))
        enc = [[e.kind, -1 if e.index is None else e.index, -1 if e.slot is None else e.slot] for e in tr]
        assert enc == json.loads(str(z[f"case{ci}"])), ci


def test_trace_documented_two_way_unrolled_shape():
    # reference test_engine.py:173-196
    plan = select_plan(3, 16, wide_backend("f32", 4).caps, unroll=2, packages=1)
    got = [(e.kind, e.index, e.slot) for e in _trace_events(plan, 16, False)]
    assert got == [
        ("init", None, None), ("load_once", None, 0), ("load_once", None, 1),
        ("load", 0, 0), ("load", 4, 1), ("vector_op", 0, 0), ("vector_op", 4, 1),
        ("store", 0, 0), ("store", 4, 1), ("load", 8, 0), ("load", 12, 1),
        ("vector_op", 8, 0), ("vector_op", 12, 1), ("store", 8, 0), ("store", 12, 1),
        ("cleanup", None, None),
    ]


def test_public_names_cover_reference_surface():
    reference_names = {
        "DenseVector", "Expression", "Leaf", "AddNode", "SubNode", "MulNode", "ScaleNode",
        "AssignNode", "SumNode", "as_node", "LengthMismatchError", "LaneVector", "LaneBackend",
        "LaneCapabilities", "scalar_backend", "wide_backend", "default_backend", "horizontal_sum",
        "CONTAINER_ALIGNMENT", "UnrollPlan", "PlanError", "select_plan", "execute_assign",
        "execute_reduce", "call_trace", "UNROLL_FACTORS", "DEFAULT_REGISTER_BUDGET", "dot", "scal",
        "axpy", "scaled_copy", "sum", "norm2", "CountingVector", "__version__",
    }
    missing = [n for n in reference_names if not hasattr(lv, n)]
    assert not missing, missing


def test_dlpack_round_trip_is_zero_copy():
    import numpy as np

    a = np.arange(10, dtype=np.float64)
    v = lv.DenseVector.from_dlpack(a)
    assert v.to_values() == list(a) and v.dtype == np.float64
    a[3] = 42.0  # shares memory
    assert v.get(3) == 42.0
    back = np.from_dlpack(v)
    assert back[3] == 42.0
    with pytest.raises(AttributeError):
        v.__cuda_array_interface__


def test_no_cuda_fails_loudly():
    """Without a CUDA device the product has no path: evaluation and the
    single-process device group raise instead of computing on the CPU."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("this process has a GPU")
    x, y = hv(np.arange(8.0)), hv(np.arange(8.0))
    with pytest.raises(RuntimeError):
        lv.DeviceGroup([0])
    with pytest.raises(RuntimeError):
        lv.dot(x, y)
    with pytest.raises(RuntimeError):
        y.assign(as_node(x) + as_node(y))


def test_assign_batch_validation_on_the_host():
    """assign_batch validates every statement before anything runs: pair
    shape, element types, lengths, and no destination shared with another
    statement (engine._check_assign_batch; no GPU needed)."""
    from paper_1109_1264_b200.engine import _check_assign_batch

    x, y, z = hv(np.arange(4.0)), hv(np.arange(4.0)), hv(np.zeros(4))
    items = _check_assign_batch([(y, as_node(y) + x), (z, as_node(x) * 2.0)])
    assert [" ".join(lw.tokens) for lw, *_ in items] == ["L0 L1 +", "S0 L0 *"]
    with pytest.raises(ValueError, match="reads the destination"):
        _check_assign_batch([(y, as_node(y) + x), (z, as_node(y) - x)])
    with pytest.raises(ValueError, match="same destination"):
        _check_assign_batch([(z, as_node(x) + y), (z, as_node(y) + x)])
    with pytest.raises(LengthMismatchError):
        _check_assign_batch([(z, as_node(x) + hv(np.arange(3.0)))])
    with pytest.raises(TypeError):
        _check_assign_batch([(z, as_node(x) + hv(np.arange(4.0), "f64"))])
    with pytest.raises(TypeError):
        _check_assign_batch([z])
