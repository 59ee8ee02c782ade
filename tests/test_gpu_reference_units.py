"""The reference's evaluating unit tests whose names are not restated
elsewhere (engine traces, bench measurement, CountingVector), with our own
cases, on the GPU path."""

import numpy as np
import pytest

import paper_1109_1264_b200 as lv
from paper_1109_1264_b200 import benchmark as sb
from paper_1109_1264_b200.engine import call_trace, masked_length
from paper_1109_1264_b200.expressions import AssignNode, ScaleNode, SumNode, as_node
from paper_1109_1264_b200.lanes import scalar_backend, wide_backend

pytestmark = pytest.mark.gpu


def dev(values, dtype="f32"):
    return lv.DenseVector.from_values(values, dtype, device="cuda")


def _bursts_ok(trace, unroll, packages):
    span = unroll // packages
    body = [e for e in trace if e.kind in ("load", "vector_op", "store")]
    assert len(body) % (3 * span) == 0
    for s in range(0, len(body), 3 * span):
        blk = body[s:s + 3 * span]
        assert [e.kind for e in blk] == ["load"] * span + ["vector_op"] * span + ["store"] * span
        loads, ops, stores = blk[:span], blk[span:2 * span], blk[2 * span:]
        assert [e.slot for e in ops] == [e.slot for e in loads] == sorted(e.slot for e in loads)
        assert [(e.index, e.slot) for e in stores] == [(e.index, e.slot) for e in loads]


@pytest.mark.parametrize("unroll", [1, 2, 4, 8])
def test_burst_order_for_every_valid_package_count(unroll):
    for packages in sorted({p for p in (1, unroll // 2, unroll) if p >= 1}):
        n = unroll * 4 * 2 + 3
        x, y = dev(np.arange(n, dtype=float)), dev(np.ones(n))
        trace = call_trace(AssignNode(as_node(y), as_node(y) + 0.5 * as_node(x)),
                           backend=wide_backend("f32", 4), unroll=unroll, packages=packages)
        _bursts_ok(trace, unroll, packages)
        kinds = [e.kind for e in trace]
        assert kinds.count("init") == 1 and kinds.count("cleanup") == 1 and kinds.count("load_once") == unroll
        singles = [i for i, k in enumerate(kinds) if k == "single_op"]
        assert len(singles) == 3 and min(singles) > max(i for i, k in enumerate(kinds) if k == "store")


def test_single_op_count_equals_tail_length():
    for n in (0, 5, 16, 17, 100):
        for unroll, width in ((1, 1), (4, 2), (2, 8)):
            x = dev(np.arange(n, dtype=float))
            d = lv.DenseVector.zeros(n, "f32", device="cuda")
            be = scalar_backend("f32") if width == 1 else wide_backend("f32", width)
            trace = call_trace(AssignNode(as_node(d), ScaleNode(-1.5, as_node(x))), backend=be, unroll=unroll)
            assert sum(e.kind == "single_op" for e in trace) == n - masked_length(n, unroll, width)
            assert d.to_values() == [-1.5 * i for i in range(n)]


@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_stepped_and_block_executors_are_bit_identical(dtype):
    g = np.random.default_rng(17)
    for n in (0, 2, 33, 1000):
        x, y = dev(g.uniform(-1, 1, n), dtype), dev(g.uniform(-1, 1, n), dtype)
        a, b = lv.DenseVector.zeros(n, dtype, device="cuda"), lv.DenseVector.zeros(n, dtype, device="cuda")
        src = as_node(y) - ScaleNode(1.25, as_node(x))
        lv.execute_assign(AssignNode(as_node(a), src), unroll=2)
        lv.execute_assign(AssignNode(as_node(b), src), unroll=2, stepped=True)
        assert a.to_array().tobytes() == b.to_array().tobytes()
        r1 = lv.execute_reduce(SumNode(as_node(x) * as_node(y)), unroll=4)
        r2 = lv.execute_reduce(SumNode(as_node(x) * as_node(y)), unroll=4, stepped=True)
        assert r1.tobytes() == r2.tobytes() and type(r1) is type(r2)


def test_trace_matches_documented_two_way_unrolled_shape():
    x = dev(np.arange(8.0))
    d = lv.DenseVector.zeros(8, "f32", device="cuda")
    trace = call_trace(AssignNode(as_node(d), ScaleNode(0.5, as_node(x))), backend=wide_backend("f32", 2),
                       unroll=2, packages=1)
    got = [(e.kind, e.index, e.slot) for e in trace]
    body = []
    for base in (0, 4):
        for kind in ("load", "vector_op", "store"):
            body += [(kind, base, 0), (kind, base + 2, 1)]
    assert got == [("init", None, None), ("load_once", None, 0), ("load_once", None, 1)] + body + \
        [("cleanup", None, None)]
    assert d.to_values() == [0.5 * i for i in range(8)]


# ---- bench
@pytest.mark.parametrize("op", ["dot", "axpy"])
def test_measure_produces_consistent_records(op):
    r = sb.measure(op, "engine", 77, "f32", 3, 1, 0)
    assert (r.op, r.variant, r.type, r.n, r.reps) == (op, "engine", "f32", 77, 3)
    assert 0 < r.best_s <= r.median_s
    assert r.gflops == sb.flop_count(op, 77) / r.best_s / 1e9
    assert r.gbytes == sb.bytes_moved(op, 77, "f32") / r.best_s / 1e9


def test_run_sweep_record_count_is_the_product():
    recs = sb.run_sweep(["dot", "scal"], ["engine", "naive"], [9, 33, 100], reps=1, warmup=0)
    assert len(recs) == 12 and len({(r.op, r.variant, r.n) for r in recs}) == 12


def test_all_variants_run():
    recs = sb.run_sweep(["scal"], list(sb.VARIANTS), [64], reps=1, warmup=0)
    assert [r.variant for r in recs] == list(sb.VARIANTS)


def test_seeded_data_is_reproducible():
    import paper_1109_1264_b200.benchmark as bm

    x1, _, _ = bm._make_data("scal", 50, np.dtype(np.float64), 3)
    x2, _, _ = bm._make_data("scal", 50, np.dtype(np.float64), 3)
    x3, _, _ = bm._make_data("scal", 50, np.dtype(np.float64), 4)
    assert x1.to_array().tobytes() == x2.to_array().tobytes() != x3.to_array().tobytes()


def test_cli_stdout_default(capsys):
    assert sb.main(["--op", "axpy", "--sizes", "16", "--reps", "1", "--warmup", "0", "--variants", "engine"]) == 0
    out = capsys.readouterr().out.splitlines()
    assert out[0] == sb.CSV_HEADER and len(out) == 2 and out[1].startswith("axpy,engine,f32,16,1,")


def test_inplace_ops_are_restored_between_reps():
    """scal / axpy mutate their operand; every rep starts from the same data,
    so the result after any number of reps is one application."""
    import paper_1109_1264_b200.benchmark as bm

    seen = []
    real = bm._engine_call

    def spy(op, x, y, out, alpha, options):
        call = real(op, x, y, out, alpha, options)

        def wrapped():
            seen.append((x if op == "scal" else y).to_array().copy())
            return call()
        return wrapped

    bm._engine_call = spy
    try:
        bm.measure("axpy", "engine", 40, "f64", 4, 2, 0)
    finally:
        bm._engine_call = real
    assert len(seen) == 6 and all(s.tobytes() == seen[0].tobytes() for s in seen)


# ---- CountingVector (reference oracle.py:72-181)
def test_counting_vector_counts_element_traffic():
    c = lv.CountingVector.from_values([1.0, 2.0, 3.0, 4.0], device="cuda")
    c.get(0)
    c.read_block(1, 4)
    c.set(2, 9.0)
    c.write_block(0, 2, np.array([5.0, 6.0], np.float32))
    assert (c.read_count, c.write_count) == (4, 3)
    c.reset_counts()
    assert (c.read_count, c.write_count) == (0, 0)


def test_counting_vector_len_and_dtype_pass_through():
    c = lv.CountingVector.zeros(6, "f64", device="cuda")
    assert len(c) == 6 and c.dtype == np.float64


def test_counting_vector_matches_plain_vector_results():
    g = np.random.default_rng(2)
    xs, ys = g.uniform(-1, 1, 300), g.uniform(-1, 1, 300)
    cx, cy = lv.CountingVector.from_values(xs, "f64", device="cuda"), lv.CountingVector.from_values(ys, "f64", device="cuda")
    px, py = dev(xs, "f64"), dev(ys, "f64")
    lv.axpy(0.75, cx, cy)
    lv.axpy(0.75, px, py)
    assert cy.to_array().tobytes() == py.to_array().tobytes()
    assert lv.dot(cx, cy) == lv.dot(px, py)
