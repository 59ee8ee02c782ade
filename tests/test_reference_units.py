"""The reference's unit-test names (pkg/tests/test_{lanes,vectors,expressions,
engine,bench}.py) restated against this package with our own cases — the
host-side behaviour a caller of `lanevec` relies on, checked without a GPU
(vectors on device="cpu"; nothing here evaluates a tree except the three
`call_trace` tests, marked gpu because call_trace evaluates, like the
reference's).  The evaluating
tests of the same files are restated in tests/test_gpu_ops_suite.py."""

import numpy as np
import pytest

import paper_1109_1264_b200 as lv
from paper_1109_1264_b200 import benchmark as sb
from paper_1109_1264_b200.engine import PlanError, UnrollPlan, call_trace, select_plan
from paper_1109_1264_b200.expressions import (AddNode, AssignNode, MulNode, ScaleNode, SubNode, SumNode,
                                              as_node, combine_partials)
from paper_1109_1264_b200.lanes import (CONTAINER_ALIGNMENT, LaneVector, as_dtype, default_backend,
                                        dtype_name, horizontal_sum, scalar_backend, wide_backend)

FLOATS = ["f32", "f64"]


def cpu(values, dtype="f32"):
    return lv.DenseVector.from_values(values, dtype, device="cpu")


# ---------------------------------------------------------------- lanes
def test_as_dtype_normalizes_spellings():
    for spelling, want in (("f64", np.float64), (np.float32, np.float32), (np.dtype("float64"), np.float64),
                           ("float32", np.float32)):
        assert as_dtype(spelling) == np.dtype(want)


@pytest.mark.parametrize("bad", [np.int16, "f2", np.complex64, bool, "uint8"])
def test_as_dtype_rejects_non_float_types(bad):
    with pytest.raises(TypeError):
        as_dtype(bad)


def test_dtype_name_round_trips():
    assert [dtype_name(as_dtype(n)) for n in FLOATS] == FLOATS


@pytest.mark.parametrize("dtype", FLOATS)
def test_splat_fills_every_lane(dtype):
    be = wide_backend(dtype, 8 if dtype == "f32" else 4)
    v = be.splat(-1.75)
    assert list(v) == [-1.75] * be.width and v.lane(be.width - 1) == -1.75
    assert v.lanes.dtype == as_dtype(dtype)


@pytest.mark.parametrize("dtype", FLOATS)
def test_horizontal_sum_of_splat_one_is_width(dtype):
    for width in (2, 4, 8):
        assert horizontal_sum(wide_backend(dtype, width).splat(1)) == width


def test_scalar_coercion():
    be = wide_backend("f64", 2)
    assert type(be.scalar(1)) is np.float64 and be.scalar(0.3) == 0.3
    assert be.zero_scalar() == 0.0
    for bad in ("0.3", None, [1.0]):
        with pytest.raises(TypeError):
            be.scalar(bad)


@pytest.mark.parametrize("dtype", FLOATS)
def test_load_store_round_trip_is_bit_exact(dtype):
    be = wide_backend(dtype, 4)
    region = np.array([np.pi, -0.0, 1e-40, np.inf, 7.0, -3.5, 0.125, 2.0], dtype=as_dtype(dtype))
    out = np.zeros_like(region)
    for off in (0, 4):
        be.store_aligned(out, off, be.load_aligned(region, off))
    assert out.tobytes() == region.tobytes()


def test_load_reads_the_addressed_window():
    region = np.arange(20, 36, dtype=np.float32)
    assert list(wide_backend("f32", 8).load_aligned(region, 8)) == list(range(28, 36))


def test_scalar_fallback_round_trip():
    be = scalar_backend("f64")
    region = np.array([4.5, -1.0])
    assert list(be.load_aligned(region, 1)) == [-1.0]


def test_store_touches_nothing_outside_the_window():
    be = wide_backend("f64", 2)
    region = np.full(6, 9.0)
    be.store_aligned(region, 2, be.splat(-4))
    assert list(region) == [9, 9, -4, -4, 9, 9]


@pytest.mark.parametrize("dtype", FLOATS)
def test_arithmetic_is_elementwise(dtype):
    g = np.random.default_rng(3)
    a, b = (g.standard_normal(4).astype(as_dtype(dtype)) for _ in range(2))
    va, vb = LaneVector(a.copy()), LaneVector(b.copy())
    assert (va + vb).lanes.tobytes() == (a + b).tobytes()
    assert (va - vb).lanes.tobytes() == (a - b).tobytes()
    assert (va * vb).lanes.tobytes() == (a * b).tobytes()


def test_arithmetic_allocates_instead_of_mutating():
    a = wide_backend("f32", 4).splat(2)
    _ = a + a
    _ = a * a
    assert list(a) == [2, 2, 2, 2]


@pytest.mark.parametrize("dtype", FLOATS)
def test_elementwise_results_match_across_widths(dtype):
    g = np.random.default_rng(5)
    x, y = (g.uniform(-1, 1, 8).astype(as_dtype(dtype)) for _ in range(2))
    outs = []
    for width in (1, 2, 4, 8):
        be = scalar_backend(dtype) if width == 1 else wide_backend(dtype, width)
        out = np.empty_like(x)
        for off in range(0, 8, width):
            be.store_aligned(out, off, be.load_aligned(x, off) * be.load_aligned(y, off)
                             + be.load_aligned(y, off))
        outs.append(out.tobytes())
    assert len(set(outs)) == 1


def test_horizontal_sum_small_cases():
    assert horizontal_sum(LaneVector(np.array([0.5, 0.25, 0.125, 0.125], np.float32))) == 1.0
    assert horizontal_sum(scalar_backend("f32").splat(3)) == 3


def test_backend_validation():
    for args in (("f32", 0, True), ("f32", 6, True), ("f64", 16, True), ("f32", 32, True), ("f64", 2, False)):
        with pytest.raises(ValueError):
            lv.LaneBackend(*args)


@pytest.mark.parametrize("dtype", FLOATS)
def test_capabilities_invariants(dtype):
    dt = as_dtype(dtype)
    for be in [scalar_backend(dtype)] + [wide_backend(dtype, w) for w in (2, 4) + ((8,) if dt.itemsize == 8 else (8, 16))]:
        c = be.caps
        assert c.width == be.width and (c.width == 1) == (not c.specialized)
        assert c.required_alignment == c.width * dt.itemsize <= CONTAINER_ALIGNMENT


def test_default_backend_fills_a_64_byte_block():
    for dtype in FLOATS:
        be = default_backend(dtype)
        assert be.width * as_dtype(dtype).itemsize == 64 and be.caps.specialized


# ---------------------------------------------------------------- vectors
@pytest.mark.parametrize("dtype", FLOATS)
def test_zeros(dtype):
    v = lv.DenseVector.zeros(5, dtype, device="cpu")
    assert len(v) == 5 and v.to_values() == [0] * 5 and v.dtype == as_dtype(dtype)


def test_zero_length_is_legal():
    v = lv.DenseVector.zeros(0, "f64", device="cpu")
    assert len(v) == 0 and v.to_values() == []


def test_negative_length_rejected():
    with pytest.raises(ValueError):
        lv.DenseVector.zeros(-3, device="cpu")


@pytest.mark.parametrize("dtype", FLOATS)
def test_from_values_round_trip(dtype):
    assert cpu([0.5, -8.0, 1024.0], dtype).to_values() == [0.5, -8.0, 1024.0]


def test_to_values_returns_dtype_scalars():
    for dtype, t in (("f32", np.float32), ("f64", np.float64)):
        assert all(type(x) is t for x in cpu([1, 2], dtype).to_values())


@pytest.mark.parametrize("n", [1, 17, 1000])
def test_storage_is_container_aligned(n):
    assert lv.DenseVector.zeros(n, device="cpu").address % CONTAINER_ALIGNMENT == 0


def test_many_allocations_stay_aligned():
    assert all(lv.DenseVector.zeros(n, "f64", device="cpu").address % CONTAINER_ALIGNMENT == 0
               for n in range(1, 40, 3))


def test_get_set_and_index_errors():
    v = cpu([4.0, 5.0, 6.0])
    assert v.get(2) == 6.0 and v[0] == 4.0
    v.set(0, -1.0)
    v[1] = 10.0
    assert v.to_values() == [-1.0, 10.0, 6.0]
    for bad in (3, -1, 100):
        with pytest.raises(IndexError):
            v.get(bad)
        with pytest.raises(IndexError):
            v.set(bad, 0.0)


def test_set_coerces_to_element_type():
    v = lv.DenseVector.zeros(2, "f32", device="cpu")
    v.set(1, 1.0 / 3.0)
    assert type(v.get(1)) is np.float32 and v.get(1) == np.float32(1.0 / 3.0)


def test_to_array_is_a_copy():
    v = cpu([3.0, 4.0])
    a = v.to_array()
    a[:] = 0
    assert v.to_values() == [3.0, 4.0]


def test_block_access_round_trip():
    v = lv.DenseVector.zeros(6, "f64", device="cpu")
    v.write_block(1, 4, np.array([7.0, 8.0, 9.0]))
    v.write_element(5, -1.0)
    assert list(v.read_block(0, 6)) == [0, 7, 8, 9, 0, -1] and v.read_element(2) == 8


def test_operators_build_nodes_without_computing():
    x, y = cpu([1.0, 2.0]), cpu([3.0, 4.0])
    assert isinstance(x - y, SubNode) and isinstance(x + y, AddNode) and isinstance(y * x, MulNode)
    assert all(isinstance(e, ScaleNode) for e in (0.5 * x, x * 0.5, -y, np.float32(3) * x))
    assert isinstance(0.5 * x + y * 2.0, AddNode)


def test_repr_smoke():
    assert "DenseVector" in repr(cpu([1.0]))
    assert "Add" in repr(cpu([1.0]) + cpu([2.0])) or "+" in repr(cpu([1.0]) + cpu([2.0]))


# ---------------------------------------------------------------- expressions
def test_as_node_wraps_vectors_and_passes_nodes_through():
    x = cpu([1.0])
    leaf = as_node(x)
    assert leaf.vector is x and as_node(leaf) is leaf
    with pytest.raises(TypeError):
        as_node(2.0)


def test_assignment_destination_must_be_a_leaf():
    x, y = cpu([1.0]), cpu([2.0])
    with pytest.raises(TypeError):
        AssignNode(as_node(x) + y, as_node(y))


def test_building_expressions_reads_nothing():
    x = lv.CountingVector.from_values([1.0, 2.0], device="cpu")
    _ = (x + x) * 2.0 - x * x
    assert x.read_count == 0 and x.write_count == 0


def test_combine_partials_order_is_slots_then_lanes_then_remainder():
    # each slot's lanes fold left to right, then the slots in order, then the
    # remainder: (1e8 + 1) rounds back to 1e8 in f32, so the ones vanish
    rows = [np.array([1e8, 1.0], dtype=np.float32), np.array([-1e8, 1.0], dtype=np.float32)]
    want = ((np.float32(1e8) + np.float32(1.0)) + (np.float32(-1e8) + np.float32(1.0))) + np.float32(0.5)
    got = combine_partials(rows, np.float32(0.5))
    assert got.tobytes() == want.tobytes() and got == 0.5


def test_combine_partials_small_case():
    assert combine_partials(np.array([[1.0, 2.0, 3.0]]), np.float64(4.0)) == 10.0


def test_combine_partials_with_no_rows_returns_remainder():
    assert combine_partials(np.zeros((0, 4), np.float32), np.float32(2.5)) == 2.5


def test_common_length_agreement_and_mismatch():
    x, y = cpu([1.0, 2.0]), cpu([3.0, 4.0])
    assert lv.common_length(AssignNode(as_node(y), as_node(x) + y)) == 2
    with pytest.raises(lv.LengthMismatchError):
        lv.common_length(AssignNode(as_node(cpu([0.0])), as_node(x) + y))


def test_mixed_element_types_rejected_at_construction():
    with pytest.raises(TypeError):
        cpu([1.0], "f32") + cpu([1.0], "f64")


def test_operator_sugar_builds_the_expected_tree():
    a, b, c = cpu([1.0]), cpu([2.0]), cpu([3.0])
    t = a - (b + c) * 3.0
    assert isinstance(t, SubNode) and isinstance(t.right, ScaleNode) and isinstance(t.right.child, AddNode)
    assert t.left.vector is a


def test_register_footprints():
    a, b = cpu([1.0]), cpu([2.0])
    assert as_node(a).register_footprint == 1
    assert (a + b).register_footprint == 2
    assert (2.0 * (a - b)).register_footprint == 3


def test_scalar_plus_vector_is_rejected():
    x = cpu([1.0])
    with pytest.raises(TypeError):
        _ = 1.0 + x
    with pytest.raises(TypeError):
        _ = 2 - x


def test_scale_alpha_is_coerced_to_element_type():
    assert type((0.1 * cpu([1.0], "f32")).alpha) is np.float32
    assert type((0.1 * cpu([1.0], "f64")).alpha) is np.float64


# ---------------------------------------------------------------- engine: plans and traces
def test_select_plan_picks_largest_fitting_unroll():
    caps = wide_backend("f64", 2).caps
    assert [select_plan(fp, 64, caps).unroll for fp in (1, 2, 3, 5, 9, 16, 40)] == [8, 8, 4, 2, 1, 1, 1]


def test_select_plan_fallback_backend_degenerates():
    p = select_plan(3, 13, scalar_backend("f64").caps)
    assert (p.unroll, p.width, p.masked_length) == (1, 1, 13)


def test_select_plan_honors_explicit_overrides():
    p = select_plan(3, 50, wide_backend("f32", 8).caps, unroll=2, packages=2)
    assert (p.unroll, p.packages, p.masked_length) == (2, 2, 48)


def test_select_plan_rejects_bad_configs():
    caps = wide_backend("f64", 4).caps
    for kw in (dict(unroll=5), dict(unroll=32), dict(unroll=8, packages=3), dict(unroll=1, packages=2)):
        with pytest.raises(PlanError):
            select_plan(2, 10, caps, **kw)
    with pytest.raises(PlanError):
        select_plan(0, 10, caps)
    with pytest.raises(PlanError):
        select_plan(1, -5, caps)


def test_root_type_guards():
    x, y = cpu([1.0]), cpu([2.0])
    with pytest.raises(TypeError):
        lv.execute_assign(SumNode(as_node(x) * y))
    with pytest.raises(TypeError):
        lv.execute_reduce(AssignNode(as_node(y), as_node(x)))


def test_backend_dtype_must_match_tree():
    x, y = cpu([1.0] * 4, "f32"), cpu([1.0] * 4, "f32")
    with pytest.raises(PlanError):
        lv.execute_assign(AssignNode(as_node(y), as_node(y) + x), backend=wide_backend("f64", 2))


def test_prebuilt_plan_is_validated_against_tree_and_backend():
    x, y = cpu([1.0] * 8), cpu([1.0] * 8)
    root = AssignNode(as_node(y), as_node(y) + 2.0 * as_node(x))
    with pytest.raises(PlanError):
        lv.execute_assign(root, UnrollPlan(2, 8, 1, 16), backend=wide_backend("f32", 4))


@pytest.mark.gpu  # call_trace evaluates the tree, as the reference's does
def test_trace_unroll_one_degenerates_to_load_op_store():
    x, d = cpu(range(6)), lv.DenseVector.zeros(6, device="cpu")
    kinds = [e.kind for e in call_trace(AssignNode(as_node(d), as_node(x)), backend=wide_backend("f32", 2),
                                        unroll=1)]
    assert kinds == ["init", "load_once"] + ["load", "vector_op", "store"] * 3 + ["cleanup"]


@pytest.mark.gpu
def test_trace_zero_length_still_brackets_with_init_and_cleanup():
    x, d = lv.DenseVector.zeros(0, device="cpu"), lv.DenseVector.zeros(0, device="cpu")
    kinds = [e.kind for e in call_trace(AssignNode(as_node(d), as_node(x)), backend=wide_backend("f32", 4),
                                        unroll=2)]
    assert kinds == ["init", "load_once", "load_once", "cleanup"]


@pytest.mark.gpu
def test_reduction_trace_ends_with_reduction_event():
    x = cpu(range(8))
    trace = call_trace(SumNode(as_node(x) * x), backend=wide_backend("f32", 4), unroll=1)
    assert trace[-1].kind == "reduction" and trace[0].kind == "init"


# ---------------------------------------------------------------- bench
def test_flop_and_byte_accounting():
    assert [sb.flop_count(op, 8) for op in ("dot", "scal", "axpy", "scaled_copy")] == [16, 8, 16, 8]
    assert [sb.bytes_moved(op, 8, "f64") for op in ("dot", "scal", "axpy", "scaled_copy")] == [128, 128, 192, 128]


def test_default_sizes_cover_powers_of_two_with_neighbors():
    sizes = sb.default_sizes()
    for p in range(6, 23):
        assert {(1 << p) - 1, 1 << p, (1 << p) + 1} <= set(sizes)
    assert sizes == sorted(set(sizes)) and sizes[-1] == (1 << 22) + 1
    big = sb.gpu_sizes()
    for p in (8, 16, 24, 28):
        assert {(1 << p) - 1, 1 << p, (1 << p) + 1} <= set(big)


def test_emit_csv_header_only_for_no_records(tmp_path):
    f = tmp_path / "empty.csv"
    sb.emit_csv([], str(f))
    assert f.read_text().splitlines() == [sb.CSV_HEADER]


def test_emit_csv_and_parse_round_trip(tmp_path):
    rec = sb.BenchRecord("axpy", "engine", "f64", 3, 2, 1.5e-6, 2e-6, 0.004, 0.048)
    f = tmp_path / "r.csv"
    sb.emit_csv([rec], str(f))
    assert sb.parse_csv(f.read_text()) == [rec]


def test_emit_csv_to_stdout(capsys):
    sb.emit_csv([sb.BenchRecord("dot", "naive", "f32", 1, 1, 1.0, 1.0, 2.0, 8.0)], "-")
    out = capsys.readouterr().out.splitlines()
    assert out[0] == sb.CSV_HEADER and out[1].startswith("dot,naive,f32,1,1,")


def test_parse_csv_rejects_bad_header():
    with pytest.raises(ValueError):
        sb.parse_csv("a,b,c\n1,2,3\n")


def test_run_sweep_rejects_unknown_names():
    with pytest.raises(ValueError):
        sb.run_sweep(["gemm"], ["engine"], [8])
    with pytest.raises(ValueError):
        sb.run_sweep(["dot"], ["fast"], [8])


def test_cli_unwritable_csv_exits_1(tmp_path, monkeypatch):
    monkeypatch.setattr(sb, "run_sweep", lambda *a, **k: [])
    assert sb.main(["--op", "dot", "--sizes", "8", "--csv", str(tmp_path / "no" / "such" / "dir.csv")]) == 1


def test_cli_writes_csv(tmp_path, monkeypatch):
    rec = sb.BenchRecord("dot", "engine", "f32", 8, 1, 1e-6, 1e-6, 0.016, 0.064)
    monkeypatch.setattr(sb, "run_sweep", lambda *a, **k: [rec])
    f = tmp_path / "o.csv"
    assert sb.main(["--op", "dot", "--sizes", "8", "--csv", str(f)]) == 0
    assert sb.parse_csv(f.read_text()) == [rec]


def test_simd_available_reports_backend_capability():
    assert sb.simd_available("f32") == default_backend("f32").caps.specialized


def test_cli_cache_sizes_sidecar(tmp_path, monkeypatch):
    monkeypatch.setattr(sb, "run_sweep", lambda *a, **k: [])
    f = tmp_path / "c.csv"
    assert sb.main(["--op", "dot", "--sizes", "8", "--csv", str(f), "--cache-sizes", "49152,2097152"]) == 0
    assert (tmp_path / "c.csv.meta").read_text() == "cache_sizes_bytes,49152,2097152\n"


def test_cli_cache_sizes_ignored_on_stdout(capsys, monkeypatch):
    monkeypatch.setattr(sb, "run_sweep", lambda *a, **k: [])
    assert sb.main(["--op", "dot", "--sizes", "8", "--cache-sizes", "1024"]) == 0
    assert "ignored" in capsys.readouterr().err
