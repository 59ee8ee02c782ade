"""The postfix interpreter kernel (csrc/salt_interp.cuh): the fallback for
trees that are neither compiled in nor JIT-compilable (no NVRTC), forced
here with salt_set_force_interp.  Elementwise results must be the
reference's bits, exactly as from the template kernels; reductions within
the BASELINE tolerance of the exact sum."""

import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

import paper_1109_1264_b200 as lv
from conftest import NP, same_bits
from oracle import restate
from paper_1109_1264_b200 import _native
from paper_1109_1264_b200.engine import execute_reduce
from paper_1109_1264_b200.expressions import SumNode, as_node, lower
from test_gpu_random_trees import random_tree

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]
TOL = {"f32": 1e-5, "f64": 1e-12}


@pytest.fixture
def interp():
    lib = _native.lib()
    lib.salt_set_force_interp(1)
    yield lib
    lib.salt_set_force_interp(0)


@pytest.mark.parametrize("dt", ["f32", "f64"])
def test_interpreter_random_trees(interp, dt):
    rng = np.random.default_rng(4242 if dt == "f32" else 4243)
    before = interp.salt_interp_launch_count()
    checked = 0
    for case in range(24):
        n = int(rng.choice([1, 7, 33, 1000, 4099, 65_537, 1 << 20]))
        nv = int(rng.integers(1, 9))
        host = [rng.uniform(-2, 2, n).astype(NP[dt]) for _ in range(nv)]
        vecs = [lv.DenseVector.from_values(h, dt, device="cuda") for h in host]
        expr = as_node(random_tree(rng, vecs, int(rng.integers(1, 7))))
        lw = lower(expr)
        idx = [next(i for i, v in enumerate(vecs) if v is u) for u in lw.vectors]
        want = restate.eval_sig(" ".join(lw.tokens), [host[i] for i in idx], lw.scalars, dt)
        out = lv.DenseVector.zeros(n, dt, device="cuda")
        out.assign(expr)
        assert same_bits(out.to_array(), want), (case, " ".join(lw.tokens))
        r = execute_reduce(SumNode(expr))
        exact = restate.exact_sum(want)
        if exact != 0 and np.isfinite(exact):
            scale = restate.exact_sum(np.abs(want))
            assert abs(float(r) - exact) <= TOL[dt] * max(abs(exact), 1e-3 * scale), (case, float(r), exact)
        # the interpreter walks the compiled kernel's tiles in its order:
        # the reduction has the compiled (table or JIT) kernel's bits
        interp.salt_set_force_interp(0)
        r_compiled = execute_reduce(SumNode(expr))
        interp.salt_set_force_interp(1)
        assert same_bits(np.array([r]), np.array([r_compiled])), (case, float(r), float(r_compiled))
        checked += 1
    assert checked == 24
    assert interp.salt_interp_launch_count() - before >= 48


@pytest.mark.parametrize("dt", ["f32", "f64"])
def test_interpreter_baseline_trees_and_misaligned_views(interp, dt):
    """Config 2's T2 and config 4's e-tree, on aligned vectors and on views
    at every element offset of a 32-byte vector (head / V = 1 paths)."""
    rng = np.random.default_rng(5)
    n = 100_003
    host = [rng.uniform(-1, 1, n + 8).astype(NP[dt]) for _ in range(4)]
    base = [lv.DenseVector.from_values(h, dt, device="cuda") for h in host]
    for off in range(0, 8 if dt == "f32" else 4):
        a, b, c, d = (lv.DenseVector.from_tensor(v.tensor[off:off + n]) for v in base)
        ha, hb, hc, hd = (h[off:off + n] for h in host)
        out = lv.DenseVector.zeros(n, dt, device="cuda")
        out.assign(1.25 * a + -0.75 * (b - c))
        want = restate.eval_sig("S0 L0 * S1 L1 L2 - * +", [ha, hb, hc], [1.25, -0.75], dt)
        assert same_bits(out.to_array(), want), off
        out.assign(1.25 * (a + b) - 0.75 * (c - d) + 0.5 * a)
        want = restate.eval_sig("S0 L0 L1 + * S1 L2 L3 - * - S2 L0 * +", [ha, hb, hc, hd],
                                [1.25, 0.75, 0.5], dt)
        assert same_bits(out.to_array(), want), off


def test_interpreter_fused_statements_device_scalars_and_axpy_dot(interp):
    _fused_sequence(interp, check=True)


def _fused_sequence(lib, check):
    n = 300_001
    g = np.random.default_rng(9)
    x, p, r, q = (g.standard_normal(n) for _ in range(4))
    X, P, R, Q = (lv.DenseVector.from_values(v, "f64") for v in (x, p, r, q))
    al = lv.DeviceScalar.full(0.375, "f64", device="cuda")
    rr = lv.fused((X, X + al * P), (R, R - al * Q), R * R)
    x1 = restate.eval_sig("L0 S0 L1 * +", [x, p], [0.375], "f64")
    r1 = restate.eval_sig("L0 S0 L1 * -", [r, q], [0.375], "f64")
    assert X.to_array().tobytes() == x1.tobytes() and R.to_array().tobytes() == r1.tobytes()
    ex = restate.exact_sum(r1 * r1)
    assert abs(float(rr) - ex) <= 1e-12 * abs(ex)
    z = g.standard_normal(n)
    Z = lv.DenseVector.from_values(z, "f64")
    s = lv.axpy_dot(0.5, P, X, Z)
    x2 = restate.eval_sig("L0 S0 L1 * +", [x1, p], [0.5], "f64")
    assert X.to_array().tobytes() == x2.tobytes()
    ex = restate.exact_sum(x2 * z)
    assert abs(float(s) - ex) <= 1e-12 * abs(ex)
    assert float(lv.dot(lv.DenseVector.zeros(0, "f64"), lv.DenseVector.zeros(0, "f64"))) == 0.0
    return float(rr), float(s)


def test_interpreter_reductions_match_compiled_bits(interp):
    """Fused statements + reduction and fused axpy->dot: the same bits on
    the interpreter and on the compiled kernels."""
    got = _fused_sequence(interp, check=True)
    interp.salt_set_force_interp(0)
    want = _fused_sequence(interp, check=True)
    interp.salt_set_force_interp(1)
    assert got == want
    # sizes across every grid shape: one CTA, one cluster (3-32 tiles), one
    # group, two ticket levels
    for dt, n in (("f32", 1 << 22), ("f64", 1 << 22), ("f32", 12345), ("f64", 3), ("f64", 1 << 16),
                  ("f32", 1 << 17), ("f64", 1 << 25)):
        g = np.random.default_rng([n, len(dt)])
        x, y = (lv.DenseVector.from_values(g.standard_normal(n), dt) for _ in range(2))
        a = (lv.dot(x, y), lv.norm2(x), lv.sum(x))
        interp.salt_set_force_interp(0)
        b = (lv.dot(x, y), lv.norm2(x), lv.sum(x))
        interp.salt_set_force_interp(1)
        assert same_bits(np.array(a), np.array(b)), (dt, n, a, b)


def test_interpreter_refuses_programs_beyond_its_shared_memory(interp):
    import torch

    deep = " ".join(["L0"] * 30) + " +" * 29   # 30-deep right-leaning stack
    x = torch.ones(64, dtype=torch.float64, device="cuda")
    out = torch.empty(64, dtype=torch.float64, device="cuda")
    leaves, keep = _native.ptr_array([x.data_ptr()])
    sc, keep2 = _native.double_array([])
    rc = interp.salt_assign(1, deep.encode(), out.data_ptr(), leaves, 1, sc, 0, 64, None)
    assert rc == -3 and b"interpreter slots" in interp.salt_last_error()


def test_without_nvrtc_out_of_table_trees_fall_back_to_the_interpreter():
    """SALT_NO_JIT=1 makes the library behave as if NVRTC were absent: an
    out-of-table tree runs on the interpreter (same bits), an in-table tree
    still on its compiled kernel."""
    code = r"""
import numpy as np, paper_1109_1264_b200 as lv
from paper_1109_1264_b200 import _native
from oracle import restate
lib = _native.lib()
g = np.random.default_rng(1)
a, b, c = (g.uniform(-1, 1, 5000) for _ in range(3))
A, B, C = (lv.DenseVector.from_values(v, "f64") for v in (a, b, c))
D = lv.DenseVector.zeros(5000, "f64")
k0 = lib.salt_interp_launch_count()
D.assign(A * B + C * A - B)                       # not in the compiled-in table
want = restate.eval_sig("L0 L1 * L2 L0 * + L1 -", [a, b, c], [], "f64")
assert D.to_array().tobytes() == want.tobytes()
k1 = lib.salt_interp_launch_count()
D.assign(A + (B - C))                             # config 2 T1: compiled in
assert lib.salt_interp_launch_count() == k1 and k1 == k0 + 1
print("ok")
"""
    env = dict(os.environ, SALT_NO_JIT="1", PYTHONPATH=f"{ROOT}:{ROOT / 'tests'}")
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env,
                         cwd=ROOT, timeout=300)
    assert out.returncode == 0 and out.stdout.strip().endswith("ok"), out.stderr[-3000:]


def test_tiered_jit_interpreter_first_then_compiled():
    """A tree outside the table and the (here disabled) disk cache: the
    first calls run on the interpreter without waiting for NVRTC; once the
    background compile is done the compiled kernel takes over — same bits
    for the assignment and for the reduction throughout."""
    code = r"""
import time, numpy as np, paper_1109_1264_b200 as lv
from paper_1109_1264_b200 import _native
from oracle import restate
lib = _native.lib()
g = np.random.default_rng(2)
a, b, c, d = (g.uniform(-1, 1, 1 << 20) for _ in range(4))
A, B, C, Dv = (lv.DenseVector.from_values(v, "f64") for v in (a, b, c, d))
E = lv.DenseVector.zeros(1 << 20, "f64")
k0 = lib.salt_interp_launch_count()
t = time.perf_counter()
E.assign((A - B) * (C + Dv) - 0.5 * A)            # fresh tree: interpreter now, NVRTC in the background
r1 = lv.dot(E - C, Dv)                            # fresh reduction tree
first_ms = (time.perf_counter() - t) * 1e3
assert lib.salt_interp_launch_count() == k0 + 2
want = restate.eval_sig("L0 L1 - L2 L3 + * S0 L0 * -", [a, b, c, d], [0.5], "f64")
e1 = E.to_array()
assert e1.tobytes() == want.tobytes()
assert lib.salt_jit_wait() == 0
k1 = lib.salt_interp_launch_count()
E.assign((A - B) * (C + Dv) - 0.5 * A)
r2 = lv.dot(E - C, Dv)
assert lib.salt_interp_launch_count() == k1       # compiled kernels now
assert E.to_array().tobytes() == e1.tobytes() and r1.tobytes() == r2.tobytes()
print("ok first_ms=%.1f" % first_ms)
"""
    env = dict(os.environ, SALT_JIT_CACHE="off", SALT_JIT_ASYNC="1", PYTHONPATH=f"{ROOT}:{ROOT / 'tests'}")
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env,
                         cwd=ROOT, timeout=300)
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr[-3000:]
    first_ms = float(out.stdout.split("first_ms=")[1])
    assert first_ms < 300, first_ms   # a synchronous NVRTC build alone takes ~400 ms per tree


def test_tiered_jit_under_concurrent_threads():
    """Eight host threads evaluate fresh trees while the background JIT
    compiles them (tiered JIT on, in a child process): every result has the
    reference's bits, before and after the compiled kernels take over."""
    code = r"""
import threading, numpy as np, torch, paper_1109_1264_b200 as lv
from paper_1109_1264_b200.expressions import as_node
from oracle import restate
n = 50_003
g = np.random.default_rng(77)
host = [g.uniform(-1, 1, n) for _ in range(4)]
vecs = [lv.DenseVector.from_values(h, "f64") for h in host]
errors = []
def work(t):
    try:
        torch.cuda.set_device(0)
        s = torch.cuda.Stream()
        c = 0.25 * (t + 1)
        with torch.cuda.stream(s):
            out = lv.DenseVector.zeros(n, "f64")
            want = restate.eval_sig("L0 S0 * L1 - L2 L3 S1 * + *", host, [c, c], "f64")
            for _ in range(20):
                out.assign((as_node(vecs[0]) * c - vecs[1]) * (as_node(vecs[2]) + vecs[3] * c))
                s.synchronize()
                if out.to_array().tobytes() != want.tobytes():
                    errors.append(t)
                    return
    except Exception as exc:
        errors.append(repr(exc))
threads = [threading.Thread(target=work, args=(t,)) for t in range(8)]
for th in threads: th.start()
for th in threads: th.join()
assert not errors, errors
lv.jit_wait()
print("ok")
"""
    env = dict(os.environ, SALT_JIT_CACHE="off", SALT_JIT_ASYNC="1", PYTHONPATH=f"{ROOT}:{ROOT / 'tests'}")
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env,
                         cwd=ROOT, timeout=300)
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr[-3000:]


def test_interpreter_on_pinned_host_vectors(interp):
    """Host vectors stream through the GPU in chunks (salt_*_host); the
    interpreter runs each chunk with the same bits."""
    n = (1 << 21) + 3
    g = np.random.default_rng(21)
    a, b, c = (g.uniform(-1, 1, n) for _ in range(3))
    A, B, C = (lv.DenseVector.from_values(v, "f64", device="cpu") for v in (a, b, c))
    D = lv.DenseVector.zeros(n, "f64", device="cpu")
    k0 = interp.salt_interp_launch_count()
    D.assign(1.25 * A + -0.75 * (B - C))
    want = restate.eval_sig("S0 L0 * S1 L1 L2 - * +", [a, b, c], [1.25, -0.75], "f64")
    assert D.to_array().tobytes() == want.tobytes()
    r = lv.dot(A, B)
    ex = restate.exact_sum(a * b)
    assert abs(float(r) - ex) <= 1e-12 * abs(ex)
    assert interp.salt_interp_launch_count() > k0


def test_fresh_tree_captured_in_a_graph_without_warm_up():
    """A tree never seen before, first evaluated inside CUDA-graph capture:
    the capture builds it synchronously (a graph must not keep the
    interpreter kernel), and replays give the reference's bits."""
    import torch

    n = 100_003
    g = np.random.default_rng(99)
    a, b, c = (g.uniform(-1, 1, n) for _ in range(3))
    A, B, C = (lv.DenseVector.from_values(v, "f64") for v in (a, b, c))
    D = lv.DenseVector.zeros(n, "f64")
    lib = _native.lib()
    k0 = lib.salt_interp_launch_count()
    s = torch.cuda.Stream()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=s):
        D.assign((A * 0.8125 - B) * (C - A * 0.4375))   # out-of-table, fresh
    graph.replay()
    graph.replay()
    torch.cuda.synchronize()
    want = restate.eval_sig("L0 S0 * L1 - L2 L0 S1 * - *", [a, b, c], [0.8125, 0.4375], "f64")
    assert D.to_array().tobytes() == want.tobytes()
    assert lib.salt_interp_launch_count() == k0   # the compiled kernel was captured
