"""Single-process multi-GPU (DeviceGroup, salt_allreduce_sum; SURVEY.md
§8(b)/(e)).  This pool has one GPU per box, so the NCCL path runs with
G = 1 here; the multi-device cases run where torch sees >= 2 GPUs.  The
fold over G partials is the same finish kernel the G-rank emulation in
test_gpu_configs.py exercises for G = 1..8."""

import ctypes

import numpy as np
import pytest
import torch

import paper_1109_1264_b200 as lv
from oracle import restate
from paper_1109_1264_b200 import _native

pytestmark = pytest.mark.gpu

TOL = {"f64": 1e-12, "f32": 1e-5}


def _vals(seed, n):
    return np.random.default_rng([1109, seed, n]).standard_normal(n)


@pytest.mark.parametrize("dt", ["f64", "f32"])
@pytest.mark.parametrize("n", [0, 1, 1000, 100_003, 1 << 22])
def test_devicegroup_dot_norm2_one_device(dt, n):
    x, y = _vals(1, n), _vals(2, n)
    npdt = np.float64 if dt == "f64" else np.float32
    xt, yt = x.astype(npdt), y.astype(npdt)
    with lv.DeviceGroup([0]) as dg:
        xs, ys = dg.scatter(x, dt), dg.scatter(y, dt)
        r = dg.dot(xs, ys)
        q = dg.norm2(xs)
        assert r.dtype == npdt and q.dtype == npdt
        ex = restate.exact_sum((xt * yt).astype(np.float64)) if n else 0.0
        exq = np.sqrt(restate.exact_sum((xt * xt).astype(np.float64))) if n else 0.0
        assert abs(float(r) - ex) <= TOL[dt] * abs(ex), (float(r), ex)
        assert abs(float(q) - exq) <= TOL[dt] * abs(exq), (float(q), exq)
        # the same bits as the ordinary single-GPU reduction of one block
        if n:
            assert r == lv.dot(xs[0], ys[0]) and q == lv.norm2(xs[0])
        lazy = dg.dot(xs, ys, lazy=True)
        assert len(lazy) == 1 and lazy[0].item() == r


def test_allreduce_abi_matches_reduce_finish_bits():
    """salt_allreduce_sum at G = 1 (NCCL all-gather of one partial + fold)
    gives the bits of salt_reduce_finish over the same partial."""
    n = 3_000_017
    X = lv.DenseVector.from_values(_vals(3, n), "f64")
    Y = lv.DenseVector.from_values(_vals(4, n), "f64")
    lib = _native.lib()
    ws = torch.zeros(lib.salt_reduce_workspace_bytes(), dtype=torch.uint8, device="cuda")
    stream = torch.cuda.current_stream().cuda_stream
    part = torch.empty(2, dtype=torch.float64, device="cuda")
    leaves, k1 = _native.ptr_array([X.tensor.data_ptr(), Y.tensor.data_ptr()])
    sc, k2 = _native.double_array([])
    _native.check(lib.salt_reduce(1, b"L0 L1 *", leaves, 2, sc, 0, n, _native.SALT_PARTIAL,
                                  ws.data_ptr(), ws.numel(), part.data_ptr(), None, stream))
    ref = torch.empty(1, dtype=torch.float64, device="cuda")
    _native.check(lib.salt_reduce_finish(1, part.data_ptr(), 1, 0, ref.data_ptr(), None, stream))
    comms = (ctypes.c_void_p * 1)()
    devs = (ctypes.c_int * 1)(0)
    _native.check(lib.salt_nccl_comm_init_all(1, ctypes.addressof(devs), ctypes.addressof(comms)))
    try:
        outs, k3 = _native.ptr_array([part.data_ptr()])
        strs, k4 = _native.ptr_array([stream])
        _native.check(lib.salt_allreduce_sum(outs, 1, 1, ctypes.addressof(comms), strs))
        torch.cuda.synchronize()
        assert part[0].item() == ref.item()
        # a communicator of the wrong size is refused before any NCCL call
        outs2, k5 = _native.ptr_array([part.data_ptr(), part.data_ptr()])
        strs2, k6 = _native.ptr_array([stream, stream])
        pair = (ctypes.c_void_p * 2)(comms[0], comms[0])
        assert lib.salt_allreduce_sum(outs2, 2, 1, ctypes.addressof(pair), strs2) == -1
        assert b"rank g" in lib.salt_last_error()
    finally:
        _native.check(lib.salt_nccl_comm_destroy(1, ctypes.addressof(comms)))
    assert comms[0] is None


def test_devicegroup_elementwise_blocks_bit_exact():
    n = 1 << 20 | 77
    a, b, c = _vals(5, n), _vals(6, n), _vals(7, n)
    with lv.DeviceGroup([0]) as dg:
        A, B, C = (dg.scatter(v, "f64") for v in (a, b, c))
        D = dg.zeros(n, "f64")
        for g in range(dg.size):
            D[g].assign(1.25 * A[g] + -0.625 * (B[g] - C[g]))
        got = dg.gather(D)
    want = restate.eval_sig("S0 L0 * S1 L1 L2 - * +", [a, b, c], [1.25, -0.625], "f64")
    assert got.tobytes() == want.tobytes()


def test_devicegroup_validation():
    with lv.DeviceGroup([0]) as dg:
        xs = dg.scatter(_vals(8, 100), "f64")
        with pytest.raises(ValueError, match="one summand per device"):
            dg.reduce([xs[0] * xs[0], xs[0] * xs[0]])
        ys = [lv.DenseVector.from_values(_vals(9, 100), "f64", device="cpu")]
        with pytest.raises(ValueError, match="DenseVector on cuda:0"):
            dg.dot(xs, ys)
    with pytest.raises(ValueError, match="distinct devices"):
        lv.DeviceGroup([0, 0])


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs >= 2 GPUs in this process")
def test_devicegroup_all_devices_agree():
    G = torch.cuda.device_count()
    n = (1 << 24) + 12345
    x, y = _vals(10, n), _vals(11, n)
    with lv.DeviceGroup(list(range(G))) as dg:
        xs, ys = dg.scatter(x, "f64"), dg.scatter(y, "f64")
        rs = dg.dot(xs, ys, lazy=True)
        vals = [r.item() for r in rs]
        assert len(set(vals)) == 1
        ex = restate.exact_sum(x * y)
        assert abs(vals[0] - ex) <= 1e-12 * abs(ex)


@pytest.mark.parametrize("dt", ["f64", "f32"])
def test_devicegroup_fused_axpy_dot_and_cg_update(dt):
    """Config 5's fused step and a CG update through DeviceGroup: the same
    bits as lv.axpy_dot / lv.fused on one device (partial + all-reduce of
    one partial == the direct finish)."""
    n = 1 << 20 | 5
    x, y, z = _vals(12, n), _vals(13, n), _vals(14, n)
    with lv.DeviceGroup([0]) as dg:
        xs, ys, zs = dg.scatter(x, dt), dg.scatter(y, dt), dg.scatter(z, dt)
        X, Y, Z = (lv.DenseVector.from_values(v, dt) for v in (x, y, z))
        for k in range(3):
            r = dg.axpy_dot(0.5, xs, ys, zs)
            q = lv.axpy_dot(0.5, X, Y, Z)
            assert r.dtype == q.dtype and r == q, (k, r, q)
            assert ys[0].to_array().tobytes() == Y.to_array().tobytes()
        a = lv.DeviceScalar.full(0.125, dt, device="cuda")
        rr = dg.fused([((xs[0], xs[0] + a * zs[0]), (ys[0], ys[0] - a * xs[0]), ys[0] * ys[0])], lazy=True)
        qq = lv.fused((X, X + a * Z), (Y, Y - a * X), Y * Y, lazy=True)
        assert rr[0].item() == qq.item()
        assert xs[0].to_array().tobytes() == X.to_array().tobytes()
        with pytest.raises(TypeError, match="expression to sum"):
            dg.fused([((xs[0], xs[0] + ys[0]),)])


def test_config5_example_runs_and_checks():
    import json
    import subprocess
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parents[1]
    out = subprocess.run([sys.executable, str(root / "examples" / "c5_devicegroup.py"), "--n", str(1 << 22),
                          "--iters", "5", "--check"], capture_output=True, text=True, timeout=300, cwd=root)
    assert out.returncode == 0, out.stderr[-3000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["checked"] is True and line["gpus"] == torch.cuda.device_count()
