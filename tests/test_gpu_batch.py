"""Batched assignments (lv.assign_batch / salt_assign_batch): many
independent trees of one shape in one launch, each result with the bits of
its own assign."""

import numpy as np
import pytest
import torch

import paper_1109_1264_b200 as lv
from oracle import restate
from paper_1109_1264_b200 import _native

pytestmark = pytest.mark.gpu


def _launches():
    return _native.lib().salt_launch_count()


@pytest.mark.parametrize("dt", ["f64", "f32"])
def test_batch_of_axpys_and_t2_trees_bit_exact(dt):
    npdt = np.float64 if dt == "f64" else np.float32
    g = np.random.default_rng([31, len(dt)])
    sts, wants, outs = [], [], []
    # 150 axpys (ragged, some misaligned views, some empty) + 70 T2 trees
    base = lv.DenseVector.from_values(g.uniform(-1, 1, 1 << 16), dt)
    for k in range(150):
        n = int(g.integers(0, 5000))
        x = g.uniform(-1, 1, n).astype(npdt)
        off = int(g.integers(0, 8)) if k % 5 == 0 else 0
        X = lv.DenseVector.from_values(x, dt)
        Y = lv.DenseVector.from_tensor(torch.empty(n + 8, dtype=X.tensor.dtype, device="cuda")[off:off + n])
        y = g.uniform(-1, 1, n).astype(npdt)
        Y.tensor.copy_(torch.from_numpy(y))
        al = float(g.uniform(-2, 2))
        sts.append((Y, lv.expressions.as_node(Y) + al * X))
        alt = npdt(al)
        wants.append(restate.eval_sig("L0 S0 L1 * +", [y, x], [float(alt)], dt))
        outs.append(Y)
    for k in range(70):
        n = int(g.integers(1, 20000))
        a, b, c = (g.uniform(-1, 1, n).astype(npdt) for _ in range(3))
        A, B, C = (lv.DenseVector.from_values(v, dt) for v in (a, b, c))
        D = lv.DenseVector.zeros(n, dt)
        al, be = float(g.uniform(-2, 2)), float(g.uniform(-2, 2))
        sts.append((D, al * A + be * (B - C)))
        wants.append(restate.eval_sig("S0 L0 * S1 L1 L2 - * +", [a, b, c],
                                      [float(npdt(al)), float(npdt(be))], dt))
        outs.append(D)
    l0 = _launches()
    done = lv.assign_batch(sts)
    launches = _launches() - l0
    assert done == 220
    assert launches <= 4, launches  # 2 shapes x ceil(count / 96)
    for k, (o, w) in enumerate(zip(outs, wants)):
        assert o.to_array().tobytes() == w.tobytes(), k
    del base


def test_batch_matches_individual_assigns_and_falls_back_beyond_limits():
    g = np.random.default_rng(8)
    n = 3000
    vs = [lv.DenseVector.from_values(g.uniform(-1, 1, n), "f64") for _ in range(10)]
    # 10 leaves > the batch limit of 8: one launch per statement, same bits
    tree = lambda k: sum((float(j + k) * vs[j] for j in range(1, 10)), start=lv.expressions.as_node(vs[0]))
    outs_b = [lv.DenseVector.zeros(n, "f64") for _ in range(3)]
    outs_i = [lv.DenseVector.zeros(n, "f64") for _ in range(3)]
    lv.assign_batch([(outs_b[k], tree(k)) for k in range(3)])
    for k in range(3):
        outs_i[k].assign(tree(k))
        assert outs_b[k].to_array().tobytes() == outs_i[k].to_array().tobytes()


def test_batch_validation():
    x = lv.DenseVector.from_values(np.arange(10.0), "f64")
    y = lv.DenseVector.from_values(np.arange(10.0), "f64")
    z = lv.DenseVector.zeros(10, "f64")
    with pytest.raises(ValueError, match="reads the destination"):
        lv.assign_batch([(y, lv.expressions.as_node(y) + x), (z, lv.expressions.as_node(y) * 2.0)])
    with pytest.raises(ValueError, match="same destination"):
        lv.assign_batch([(z, lv.expressions.as_node(x) + y), (z, lv.expressions.as_node(x) - y)])
    with pytest.raises(lv.LengthMismatchError):
        lv.assign_batch([(z, lv.expressions.as_node(x) + lv.DenseVector.zeros(3, "f64"))])
    with pytest.raises(TypeError):
        lv.assign_batch([z])
    assert lv.assign_batch([]) == 0


def test_batch_is_one_launch_for_many_small_trees():
    """256 axpys at n = 4096: one launch per 96 instead of 256 — the device
    time drops accordingly (recorded, asserted loosely)."""
    n, m = 4096, 256
    g = np.random.default_rng(4)
    X = [lv.DenseVector.from_values(g.uniform(-1, 1, n), "f64") for _ in range(m)]
    Y = [lv.DenseVector.from_values(g.uniform(-1, 1, n), "f64") for _ in range(m)]
    sts = [(y, lv.expressions.as_node(y) + 0.5 * x) for x, y in zip(X, Y)]
    lv.assign_batch(sts)
    torch.cuda.synchronize()

    def timed(fn):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(2_000_000)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        return e0.elapsed_time(e1) * 1e3

    t_batch = min(timed(lambda: lv.assign_batch(sts)) for _ in range(5))
    t_loop = min(timed(lambda: [lv.axpy(0.5, x, y) for x, y in zip(X, Y)]) for _ in range(5))
    assert t_batch < t_loop / 3, (t_batch, t_loop)
    # end to end, host included (expressions prebuilt): one C call walks,
    # checks and groups the statements
    import time

    def wall(fn):
        torch.cuda.synchronize()
        t = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        return (time.perf_counter() - t) * 1e6

    w_batch = min(wall(lambda: lv.assign_batch(sts)) for _ in range(5))
    w_loop = min(wall(lambda: [y.assign(st) for y, st in sts]) for _ in range(5))
    assert w_batch < w_loop, (w_batch, w_loop)
    print(f"256 axpys n=4096: device {t_batch:.0f} vs {t_loop:.0f} us; wall {w_batch:.0f} vs {w_loop:.0f} us")


@pytest.mark.parametrize("dt", ["f64", "f32"])
def test_reduce_batch_bits_equal_individual_reductions(dt):
    npdt = np.float64 if dt == "f64" else np.float32
    g = np.random.default_rng([41, len(dt)])
    pairs, xs = [], []
    for k in range(180):
        n = int(g.integers(0, 4000)) if k % 30 else (1 << 20) + int(g.integers(0, 9))  # a few large ones
        x, y = (g.standard_normal(n).astype(npdt) for _ in range(2))
        off = int(g.integers(1, 4)) if k % 7 == 0 else 0
        X = lv.DenseVector.from_tensor(torch.from_numpy(np.concatenate([np.zeros(off, npdt), x])).cuda()[off:])
        Y = lv.DenseVector.from_tensor(torch.from_numpy(np.concatenate([np.zeros(off, npdt), y])).cuda()[off:])
        pairs.append((X, Y))
        xs.append(X)
    l0 = _launches()
    got = lv.dot_batch(pairs)
    launches = _launches() - l0
    assert launches <= 10, launches   # 174 small ones: 2 batched launches; 6 large: one each
    want = [lv.dot(x, y) for x, y in pairs]
    assert all(a.dtype == npdt for a in got)
    assert np.array(got).tobytes() == np.array(want).tobytes()
    nr = lv.reduce_batch([lv.expressions.as_node(x) * x for x in xs], sqrt=True)
    assert np.array(nr).tobytes() == np.array([lv.norm2(x) for x in xs]).tobytes()
    assert np.array(lv.norm2_batch(xs)).tobytes() == np.array(nr).tobytes()
    lazy = lv.dot_batch(pairs[:40], lazy=True)
    assert np.array([d.item() for d in lazy]).tobytes() == np.array(want[:40]).tobytes()
    ex = restate.exact_sum(pairs[1][0].to_array().astype(np.float64) * pairs[1][1].to_array())
    assert abs(float(got[1]) - ex) <= (1e-12 if dt == "f64" else 1e-5) * max(abs(ex), 1e-30)


def test_reduce_batch_one_launch_for_many_small_dots():
    n, m = 2048, 192
    g = np.random.default_rng(9)
    pairs = [tuple(lv.DenseVector.from_values(g.uniform(-1, 1, n), "f64") for _ in range(2)) for _ in range(m)]
    lv.dot_batch(pairs)
    l0 = _launches()
    lv.dot_batch(pairs, lazy=True)
    assert _launches() - l0 == 2   # 192 problems = 2 launches of 96


def test_batches_with_special_values_match_single_calls():
    """±0, ±inf, NaN, subnormals and huge values: batched results have the
    bits of the single calls (NaN positions for NaN)."""
    specials = np.array([0.0, -0.0, np.inf, -np.inf, np.nan, 5e-324, 1e308, -1e308, 1.0, -2.5])
    g = np.random.default_rng(13)
    for dt in ("f64", "f32"):
        npdt = np.float64 if dt == "f64" else np.float32
        pairs, sts, outs_b, outs_s = [], [], [], []
        for k in range(40):
            n = int(g.integers(1, 3000))
            x = g.uniform(-1, 1, n)
            y = g.uniform(-1, 1, n)
            if k % 3 == 0:
                idx = g.integers(0, n, size=min(n, 4))
                x[idx] = g.choice(specials, size=len(idx))
            X = lv.DenseVector.from_values(x.astype(npdt), dt)
            Y = lv.DenseVector.from_values(y.astype(npdt), dt)
            pairs.append((X, Y))
            ob, os_ = lv.DenseVector.zeros(n, dt), lv.DenseVector.zeros(n, dt)
            sts.append((ob, 0.75 * lv.expressions.as_node(X) - Y))
            outs_b.append(ob)
            outs_s.append((os_, X, Y))
        got = lv.dot_batch(pairs)
        want = [lv.dot(x, y) for x, y in pairs]
        for a, b in zip(got, want):
            assert (np.isnan(a) and np.isnan(b)) or a.tobytes() == b.tobytes(), (dt, a, b)
        lv.assign_batch(sts)
        for ob, (os_, X, Y) in zip(outs_b, outs_s):
            os_.assign(0.75 * X - Y)
            a, b = ob.to_array(), os_.to_array()
            assert np.array_equal(a, b, equal_nan=True) and np.array_equal(np.signbit(a), np.signbit(b))
