"""Programmatic dependent launch (every fused kernel is launched with
programmatic stream serialization and waits on griddepcontrol.wait before
touching memory): long chains of dependent launches, with nothing but
stream order between them, must give the results of running the steps one
at a time with the host waiting in between."""

import numpy as np
import pytest
import torch

import paper_1109_1264_b200 as lv
from oracle import restate

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n", [4096, 1 << 20])
def test_chain_of_dependent_axpys_is_sequential(n):
    g = np.random.default_rng([7, n])
    x, y = g.uniform(-1, 1, n), g.uniform(-1, 1, n)
    X, Y = lv.DenseVector.from_values(x, "f64"), lv.DenseVector.from_values(y, "f64")
    steps = 500
    for k in range(steps):  # each launch reads what the previous one wrote
        lv.axpy(0.5 if k % 2 else -0.25, X, Y)
        lv.scal(1.0009765625, X)
    want_y, want_x = y.copy(), x.copy()
    for k in range(steps):
        want_y = restate.eval_sig("L0 S0 L1 * +", [want_y, want_x], [0.5 if k % 2 else -0.25], "f64")
        want_x = restate.eval_sig("S0 L0 *", [want_x], [1.0009765625], "f64")
    assert Y.to_array().tobytes() == want_y.tobytes()
    assert X.to_array().tobytes() == want_x.tobytes()


def test_reduction_to_device_scalar_to_assignment_chain():
    """dot -> device scalar -> fused update -> dot ...: every kernel depends
    on the previous one through memory (tickets, the scalar, the vector)."""
    n = 300_007
    g = np.random.default_rng(11)
    x, y = g.standard_normal(n), g.standard_normal(n)

    def run(sync):
        X, Y = lv.DenseVector.from_values(x, "f64"), lv.DenseVector.from_values(y, "f64")
        out = []
        for _ in range(60):
            r = lv.dot(X, Y, lazy=True)
            s = r / lv.dot(X, X, lazy=True)
            if sync:
                torch.cuda.synchronize()
            Y.assign(Y - s * X)
            if sync:
                torch.cuda.synchronize()
            out.append(r)
        return Y.to_array(), [v.item() for v in out]

    async_y, async_r = run(False)
    sync_y, sync_r = run(True)
    assert async_y.tobytes() == sync_y.tobytes()
    assert async_r == sync_r


def test_chain_captured_in_a_graph_matches_eager():
    n = 1 << 16
    g = np.random.default_rng(5)
    x, y = g.uniform(-1, 1, n), g.uniform(-1, 1, n)
    X, Y = lv.DenseVector.from_values(x, "f64"), lv.DenseVector.from_values(y, "f64")
    X2, Y2 = lv.DenseVector.from_values(x, "f64"), lv.DenseVector.from_values(y, "f64")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(3):  # warm-up outside capture (JIT, workspace)
            lv.axpy(0.5, X2, Y2)
            lv.dot(X2, Y2, lazy=True)
    torch.cuda.synchronize()
    X2.tensor.copy_(X.tensor)
    Y2.tensor.copy_(Y.tensor)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=s):
        for _ in range(50):
            lv.axpy(0.5, X2, Y2)
            r = lv.dot(X2, Y2, lazy=True)
            Y2.assign(Y2 - r * 1e-9 * X2)
    graph.replay()
    torch.cuda.synchronize()
    for _ in range(50):
        lv.axpy(0.5, X, Y)
        r = lv.dot(X, Y, lazy=True)
        Y.assign(Y - r * 1e-9 * X)
    assert Y2.to_array().tobytes() == Y.to_array().tobytes()


@pytest.mark.parametrize("n", [1 << 15, 1 << 17])
def test_cluster_reduction_chain(n):
    """Cluster-launched reductions (one thread-block cluster, DSMEM combine)
    feeding assignments back to back."""
    g = np.random.default_rng([3, n])
    x = g.standard_normal(n)

    def run(sync):
        X = lv.DenseVector.from_values(x, "f64")
        rs = []
        for _ in range(40):
            q = lv.norm2(X, lazy=True)
            if sync:
                torch.cuda.synchronize()
            X.assign((1.0 / q) * X + 0.001 * X)
            rs.append(q)
        return X.to_array(), [r.item() for r in rs]

    a, b = run(False), run(True)
    assert a[0].tobytes() == b[0].tobytes() and a[1] == b[1]


@pytest.mark.parametrize("dt", ["f64", "f32"])
def test_chain_over_misaligned_views_is_sequential(dt):
    """The V = 1 kernels (operands at different misalignments) load through
    L1; a chain in which every launch reads what the previous launch wrote —
    to shifted positions, i.e. from other threads, CTAs and SMs — must still
    see each write (no stale L1 line survives a launch boundary under
    programmatic dependent launch)."""
    npdt = np.float64 if dt == "f64" else np.float32
    n = (1 << 18) + 37
    g = np.random.default_rng(21)
    base = [g.uniform(-1, 1, n + 4100).astype(npdt) for _ in range(2)]
    t = [torch.from_numpy(b).cuda() for b in base]
    # X at element offset 1, Y at offset 2: mixed misalignment -> V = 1
    X = lv.DenseVector.from_tensor(t[0][1:1 + n])
    Y = lv.DenseVector.from_tensor(t[1][2:2 + n])
    # the same storage seen 4,099 elements later (another CTA's elements)
    Xs = lv.DenseVector.from_tensor(t[0][1 + 4099:1 + 4099 + n - 4099])
    Ys = lv.DenseVector.from_tensor(t[1][2:2 + n - 4099])
    hx, hy = base[0].copy(), base[1].copy()
    for k in range(200):
        al = 0.5 if k % 2 else -0.25
        lv.axpy(al, X, Y)                 # Y += al X
        hy[2:2 + n] = restate.eval_sig("L0 S0 L1 * +", [hy[2:2 + n], hx[1:1 + n]], [al], dt)
        Xs.assign(Xs + 0.125 * Ys)        # X[4099:] += Y[:n-4099] / 8 (reads the previous launch's Y)
        hx[1 + 4099:1 + n] = restate.eval_sig("L0 S0 L1 * +", [hx[1 + 4099:1 + n], hy[2:2 + n - 4099]],
                                              [0.125], dt)
    assert t[0].cpu().numpy().tobytes() == hx.tobytes()
    assert t[1].cpu().numpy().tobytes() == hy.tobytes()
