"""Randomised parity: seeded random expression trees (up to 8 distinct
leaves, repeated leaves, scalars, depth <= 6) built with the public
operators, evaluated on the GPU (compiled-in table or NVRTC JIT) and compared
bit for bit with the NumPy restatement of the reference's node semantics;
reductions of the same trees against the exact sum."""

import numpy as np
import pytest

import paper_1109_1264_b200 as lv
from conftest import NP, same_bits
from oracle import restate
from paper_1109_1264_b200 import _native
from paper_1109_1264_b200.engine import execute_reduce
from paper_1109_1264_b200.expressions import SumNode, as_node, lower

pytestmark = pytest.mark.gpu


def random_tree(rng, vecs, depth):
    """Returns (expression, postfix-builder) using only public operators."""
    if depth == 0 or rng.random() < 0.25:
        return vecs[int(rng.integers(len(vecs)))]
    kind = rng.integers(5)
    left = random_tree(rng, vecs, depth - 1)
    if kind == 3:
        alpha = float(rng.uniform(-3, 3))
        return alpha * as_node(left) if rng.random() < 0.5 else as_node(left) * alpha
    if kind == 4:
        return -as_node(left)
    right = random_tree(rng, vecs, depth - 1)
    l, r = as_node(left), as_node(right)
    return l + r if kind == 0 else (l - r if kind == 1 else l * r)


@pytest.mark.parametrize("dt", ["f32", "f64"])
def test_random_trees_bit_exact(dt):
    rng = np.random.default_rng(2026 if dt == "f32" else 2027)
    checked = 0
    for case in range(24):
        n = int(rng.choice([1, 7, 33, 1000, 4099, 65_537, 1 << 20]))
        nv = int(rng.integers(1, 9))
        host = [rng.uniform(-2, 2, n).astype(NP[dt]) for _ in range(nv)]
        vecs = [lv.DenseVector.from_values(h, dt, device="cuda") for h in host]
        expr = as_node(random_tree(rng, vecs, int(rng.integers(1, 7))))
        lw = lower(expr)
        if len(lw.vectors) > 8:
            continue
        idx = [next(i for i, v in enumerate(vecs) if v is u) for u in lw.vectors]
        want = restate.eval_sig(" ".join(lw.tokens), [host[i] for i in idx], lw.scalars, dt)
        out = lv.DenseVector.zeros(n, dt, device="cuda")
        out.assign(expr)
        assert same_bits(out.to_array(), want), (case, " ".join(lw.tokens))
        r = execute_reduce(SumNode(expr))
        # tiered JIT: the calls above may have run on the interpreter while
        # NVRTC compiled in the background; once it is done, the compiled
        # kernels must give the same bits
        assert _native.lib().salt_jit_wait() == 0
        out2 = lv.DenseVector.zeros(n, dt, device="cuda")
        out2.assign(expr)
        assert same_bits(out2.to_array(), want), (case, "compiled", " ".join(lw.tokens))
        assert same_bits(np.array([execute_reduce(SumNode(expr))]), np.array([r])), case
        exact = restate.exact_sum(want)
        if exact != 0 and np.isfinite(exact):
            tol = {"f32": 1e-5, "f64": 1e-12}[dt]
            # exact sum of the element-typed tree values; cancellation-free bound
            scale = restate.exact_sum(np.abs(want))
            assert abs(float(r) - exact) <= tol * max(abs(exact), 1e-3 * scale), (case, float(r), exact)
        checked += 1
    assert checked >= 20


def test_trees_beyond_one_kernel_are_split_bit_exactly():
    """20 distinct vectors and 40 scalars exceed one fused kernel
    (SALT_MAX_LEAVES = 16, SALT_MAX_SCALARS = 32): the engine evaluates
    subtrees into device temporaries first — same bits, since every node
    rounds to the element type anyway."""
    rng = np.random.default_rng(99)
    n = 10_001
    for dt in ("f32", "f64"):
        host = [rng.uniform(-1, 1, n).astype(NP[dt]) for _ in range(20)]
        vecs = [lv.DenseVector.from_values(h, dt, device="cuda") for h in host]
        expr = as_node(vecs[0])
        for k in range(1, 20):
            expr = float(rng.uniform(0.5, 1.5)) * expr + float(rng.uniform(-1, 1)) * as_node(vecs[k])
        lw = lower(expr)
        assert len(lw.vectors) == 20 and len(lw.scalars) == 38
        want = restate.eval_sig(" ".join(lw.tokens), host, lw.scalars, dt)
        out = lv.DenseVector.zeros(n, dt, device="cuda")
        out.assign(expr)
        assert same_bits(out.to_array(), want), dt
        r = execute_reduce(SumNode(expr))
        exact = restate.exact_sum(want)
        assert abs(float(r) - exact) <= {"f32": 1e-5, "f64": 1e-12}[dt] * abs(exact)


def random_tree_ds(rng, vecs, depth, dt):
    """Like random_tree, but half of the scalars are DeviceScalars."""
    if depth == 0 or rng.random() < 0.25:
        return vecs[int(rng.integers(len(vecs)))]
    kind = rng.integers(5)
    left = random_tree_ds(rng, vecs, depth - 1, dt)
    if kind == 3:
        alpha = float(rng.uniform(-3, 3))
        if rng.random() < 0.5:
            alpha = lv.DeviceScalar.full(alpha, dt, device="cuda")
        return alpha * as_node(left) if rng.random() < 0.5 else as_node(left) * alpha
    if kind == 4:
        return -as_node(left)
    right = random_tree_ds(rng, vecs, depth - 1, dt)
    l, r = as_node(left), as_node(right)
    return l + r if kind == 0 else (l - r if kind == 1 else l * r)


def host_signature(lw):
    """Postfix signature with every P<k> (device scalar) replaced by an S<j>
    carrying its value: the tree the oracle evaluates."""
    toks, vals = [], []
    for t in lw.tokens:
        if t[0] == "S":
            toks.append(f"S{len(vals)}")
            vals.append(lw.scalars[int(t[1:])])
        elif t[0] == "P":
            toks.append(f"S{len(vals)}")
            vals.append(float(lw.pscalars[int(t[1:])].item()))
        else:
            toks.append(t)
    return " ".join(toks), vals


@pytest.mark.parametrize("dt", ["f32", "f64"])
def test_random_trees_with_device_scalars(dt):
    """Scalars read from device memory (P<k>) give the same bits as the
    same values passed from the host; more than 8 device scalars in one tree
    (SALT_MAX_PSCALARS) are handled by splitting."""
    rng = np.random.default_rng(3030 if dt == "f32" else 3031)
    seen_p = 0
    for case in range(24):
        n = int(rng.choice([1, 33, 4099, 65_537, 1 << 20]))
        nv = int(rng.integers(1, 7))
        host = [rng.uniform(-2, 2, n).astype(NP[dt]) for _ in range(nv)]
        vecs = [lv.DenseVector.from_values(h, dt, device="cuda") for h in host]
        expr = as_node(random_tree_ds(rng, vecs, int(rng.integers(2, 8)), dt))
        lw = lower(expr)
        seen_p += len(lw.pscalars)
        idx = [next(i for i, v in enumerate(vecs) if v is u) for u in lw.vectors]
        sig, vals = host_signature(lw)
        want = restate.eval_sig(sig, [host[i] for i in idx], vals, dt)
        out = lv.DenseVector.zeros(n, dt, device="cuda")
        out.assign(expr)
        assert same_bits(out.to_array(), want), (case, " ".join(lw.tokens))
        r = execute_reduce(SumNode(expr))
        # tiered JIT: the calls above may have run on the interpreter while
        # NVRTC compiled in the background; once it is done, the compiled
        # kernels must give the same bits
        assert _native.lib().salt_jit_wait() == 0
        out2 = lv.DenseVector.zeros(n, dt, device="cuda")
        out2.assign(expr)
        assert same_bits(out2.to_array(), want), (case, "compiled", " ".join(lw.tokens))
        assert same_bits(np.array([execute_reduce(SumNode(expr))]), np.array([r])), case
        exact = restate.exact_sum(want)
        if exact != 0 and np.isfinite(exact):
            tol = {"f32": 1e-5, "f64": 1e-12}[dt]
            scale = restate.exact_sum(np.abs(want))
            assert abs(float(r) - exact) <= tol * max(abs(exact), 1e-3 * scale), (case, float(r), exact)
    assert seen_p >= 10
    # 12 device scalars in one tree: more than one kernel takes
    n = 5003
    host = [rng.uniform(-1, 1, n).astype(NP[dt]) for _ in range(3)]
    vecs = [lv.DenseVector.from_values(h, dt, device="cuda") for h in host]
    expr = as_node(vecs[0])
    for k in range(12):
        expr = lv.DeviceScalar.full(0.5 + k / 16, dt, device="cuda") * expr + as_node(vecs[k % 3])
    lw = lower(expr)
    assert len(lw.pscalars) == 12
    sig, vals = host_signature(lw)
    want = restate.eval_sig(sig, host, vals, dt)
    out = lv.DenseVector.zeros(n, dt, device="cuda")
    out.assign(expr)
    assert same_bits(out.to_array(), want)
