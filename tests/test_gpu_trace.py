"""Device-observed traces (lv.device_trace, row f4): what one GPU thread
actually executes, against the reference stepped executor's burst order
(/root/reference/pkg/src/lanevec/engine.py:209-225: per package, all slots
load, then all slots compute, then all slots store)."""

import numpy as np
import pytest

import paper_1109_1264_b200 as lv
from paper_1109_1264_b200.engine import UnrollPlan, _trace_events, masked_length
from paper_1109_1264_b200.expressions import AssignNode, SumNode, as_node

pytestmark = pytest.mark.gpu

BLOCK, V64 = 256, 4


def dev(v):
    return lv.DenseVector.from_values(v, "f64", device="cuda")


def tiles(events):
    """Split a thread's vector events into tiles: a tile starts at a load
    that follows an op (or at the first load)."""
    out, cur, seen_op = [], [], False
    for e in events:
        if e.kind == "load" and seen_op:
            out.append(cur)
            cur, seen_op = [], False
        if e.kind in ("load", "vector_op", "store"):
            cur.append(e)
            seen_op |= e.kind != "load"
    if cur:
        out.append(cur)
    return out


@pytest.mark.parametrize("n,want_unr", [
    (4 * BLOCK * V64 * 2 + 3, 1),         # small (<= 2^20 vectors): one vector per leaf per thread
    ((1 << 22) + 4 * BLOCK * V64 * 2 + 3, 2),  # beyond: two
])
def test_assign_trace_is_a_load_burst_then_ops_in_slot_order(n, want_unr):
    # whole tiles plus a 3-element tail
    g = np.random.default_rng(1)
    a, b, c = (g.standard_normal(n) for _ in range(3))
    A, B, C = dev(a), dev(b), dev(c)
    D1, D2 = lv.DenseVector.zeros(n, "f64", device="cuda"), lv.DenseVector.zeros(n, "f64", device="cuda")
    tr = lv.device_trace(AssignNode(as_node(D1), 1.5 * A + -0.5 * (B - C)))
    D2.assign(1.5 * A + -0.5 * (B - C))   # untraced kernel: same bits
    assert D1.to_array().tobytes() == D2.to_array().tobytes()
    ev = tr.events
    assert not tr.truncated and ev
    # thread 0 of CTA 0: the first tail element, then ONE tile (one tile per CTA)
    assert ev[0].kind == "single_op" and ev[0].index == n - 3
    body = [e for e in ev if e.kind != "single_op"]
    unr = sum(1 for e in body if e.kind == "load")
    assert unr == want_unr
    assert [e.kind for e in body] == ["load"] * unr + ["vector_op", "store"] * unr
    assert [e.slot for e in body[:unr]] == list(range(unr))
    assert [e.index for e in body[:unr]] == [u * BLOCK * V64 for u in range(unr)]
    assert [e.index for e in body if e.kind == "store"] == [u * BLOCK * V64 for u in range(unr)]
    # the reference's stepped executor for the same unroll: the same load
    # burst (every slot's operands in flight before any arithmetic)
    plan = UnrollPlan(width=V64, unroll=unr, packages=1, masked_length=masked_length(n, unr, V64))
    ref = _trace_events(plan, n, False)
    ref_body = [e for e in ref if e.kind in ("load", "vector_op", "store")][:3 * unr]
    assert [e.kind for e in ref_body[:unr]] == [e.kind for e in body[:unr]]
    assert [e.slot for e in ref_body[:unr]] == [e.slot for e in body[:unr]]


@pytest.mark.parametrize("n,ntiles", [
    (1 << 20, 1),                 # collector combine: one tile per streaming CTA
    ((1 << 27) + 4 * BLOCK * V64, 2),  # > 65,536 streaming CTAs (MAX_COLLECT): 2 tiles each
])
def test_reduction_trace_walks_its_tiles_then_joins_the_combine(n, ntiles):
    g = np.random.default_rng(2)
    x, y = g.standard_normal(n), g.standard_normal(n)
    X, Y = dev(x), dev(y)
    tr = lv.device_trace(SumNode(as_node(X) * as_node(Y)))
    ev = tr.events
    assert ev[-1].kind == "reduction"
    ts = tiles(ev)
    assert len(ts) == ntiles
    unr = sum(1 for e in ts[0] if e.kind == "load")
    per_tile = BLOCK * unr * V64
    for t, tile in enumerate(ts):
        loads = [e for e in tile if e.kind == "load"]
        ops = [e for e in tile if e.kind == "vector_op"]
        assert [e.kind for e in tile] == ["load"] * unr + ["vector_op"] * unr  # burst, no stores
        assert [e.index for e in loads] == [t * per_tile + u * BLOCK * V64 for u in range(unr)]
        assert [e.index for e in ops] == [e.index for e in loads]
    # traced and untraced reductions: the same bits
    assert np.float64(tr.result).tobytes() == np.float64(lv.dot(X, Y)).tobytes()


def test_device_trace_rejects_host_vectors():
    X = lv.DenseVector.from_values(np.ones(8), "f64", device="cpu")
    with pytest.raises(TypeError):
        lv.device_trace(SumNode(as_node(X) * as_node(X)))
