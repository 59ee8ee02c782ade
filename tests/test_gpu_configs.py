"""BASELINE.json configs at their full sizes on one B200, checked against the
oracle (bit-exact elementwise; reductions vs the binary128 exact oracle with
1e-12 / 1e-5 relative tolerance), plus size-independent properties.

Inputs are the seeded chunk-keyed synthetic streams of synth.py (the same
bench.py uses).  Multi-GPU configs (4, 5) run here as one GPU's block of the
sharded problem plus an on-device emulation of the G-way partition (each
block evaluated separately, partials combined with salt_reduce_finish) —
no ranks wait on one another on a single GPU.
"""

import os

import numpy as np
import pytest
import torch

import paper_1109_1264_b200 as lv
from conftest import same_bits
from oracle import coracle, restate
from paper_1109_1264_b200 import _native, synth
from paper_1109_1264_b200.sharding import shard_bounds

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

THREADS = max(1, min(32, len(os.sched_getaffinity(0))))
TOL = {np.float32: 1e-5, np.float64: 1e-12}


def host_and_dev(cfg, operand, n, dt, lo=0):
    h = synth.block(cfg, operand, lo, lo + n, dt)
    return h, lv.DenseVector.from_values(h, np.dtype(dt), device="cuda")


def test_config1_daxpy_2p20_bit_exact():
    n = 1 << 20
    x, X = host_and_dev(1, 0, n, np.float64)
    y, Y = host_and_dev(1, 1, n, np.float64)
    (alpha,) = synth.scalars(1, 1)
    lv.axpy(alpha, X, Y)
    want = restate.eval_sig("L0 S0 L1 * +", [y, x], [alpha], "f64")
    assert Y.to_array().tobytes() == want.tobytes()


@pytest.mark.parametrize("logn", [10, 12, 14, 16, 18, 20, 22, 24, 26, 28])
def test_config2_fused_sweep_bit_exact(logn):
    n = 1 << logn
    a, A = host_and_dev(2, 0, n, np.float64)
    b, B = host_and_dev(2, 1, n, np.float64)
    c, C = host_and_dev(2, 2, n, np.float64)
    alpha, beta = synth.scalars(2, 2)
    D = lv.DenseVector.empty(n, "f64", device="cuda")
    want = np.empty(n)
    D.assign(A + (B - C))
    coracle.assign("L0 L1 L2 - +", want, [a, b, c], [], threads=THREADS)
    assert D.to_array().tobytes() == want.tobytes()
    D.assign(alpha * A + beta * (B - C))
    coracle.assign("S0 L0 * S1 L1 L2 - * +", want, [a, b, c], [alpha, beta], threads=THREADS)
    assert D.to_array().tobytes() == want.tobytes()


@pytest.mark.parametrize("dt", [np.float32, np.float64])
@pytest.mark.parametrize("logn", [24, 28])
def test_config3_reductions_vs_exact(dt, logn):
    n = 1 << logn
    x, X = host_and_dev(3, 0, n, dt)
    y, Y = host_and_dev(3, 1, n, dt)
    r = lv.dot(X, Y)
    ex = coracle.reduce_exact("L0 L1 *", [x, y], [], dt, threads=THREADS)
    assert type(r) is dt
    assert abs(float(r) - ex) <= TOL[dt] * abs(ex), (float(r), ex)
    nr = lv.norm2(X)
    exn = np.sqrt(coracle.reduce_exact("L0 L0 *", [x], [], dt, threads=THREADS))
    assert abs(float(nr) - exn) <= TOL[dt] * exn, (float(nr), exn)
    # deterministic run to run
    assert lv.dot(X, Y).tobytes() == r.tobytes()
    assert lv.norm2(X).tobytes() == nr.tobytes()


def test_config4_etree_f32_2p30_and_partitions():
    """e = alpha(a+b) - beta(c-d) + gamma*a, f32, n = 2^30: the whole vector on
    one GPU bit-exact vs the oracle, and every G in {2,4,8} block partition
    (each block evaluated as its own launch) identical to it."""
    n = 1 << 30
    dt = np.float32
    hs, ds = [], []
    for k in range(4):
        h, d = host_and_dev(4, k, n, dt)
        hs.append(h)
        ds.append(d)
    al, be, ga = synth.scalars(4, 3)
    E = lv.DenseVector.empty(n, "f32", device="cuda")
    E.assign(al * (ds[0] + ds[1]) - be * (ds[2] - ds[3]) + ga * ds[0])
    want = np.empty(n, dtype=dt)
    coracle.assign("S0 L0 L1 + * S1 L2 L3 - * - S2 L0 * +", want, hs, [al, be, ga], threads=THREADS)
    got = E.to_array()
    assert got.tobytes() == want.tobytes()
    del want, hs
    for G in (2, 4, 8):
        F = torch.empty(n, dtype=torch.float32, device="cuda")
        for r in range(G):
            lo, hi = shard_bounds(n, G, r)
            v = [lv.DenseVector.from_tensor(d.tensor[lo:hi]) for d in ds]
            f = lv.DenseVector.from_tensor(F[lo:hi])
            f.assign(al * (v[0] + v[1]) - be * (v[2] - v[3]) + ga * v[0])
        assert torch.equal(F.view(torch.int32), E.tensor.view(torch.int32)), G
        del F


def test_config5_axpy_dot_100_iterations():
    """y = alpha*x + y; r = dot(y, z), 100 iterations, f64, one GPU's block
    (2^28 = 2^31 / 8) of config 5: y bit-exact after 100 fused steps, r
    within 1e-12 of the exact value at sampled iterations."""
    n = 1 << 28
    x, X = host_and_dev(5, 0, n, np.float64)
    y, Y = host_and_dev(5, 1, n, np.float64)
    z, Z = host_and_dev(5, 2, n, np.float64)
    (alpha,) = synth.scalars(5, 1)
    rs = []
    for it in range(100):
        rs.append(lv.axpy_dot(alpha, X, Y, Z, lazy=True))
    yh = y.copy()
    for it in range(100):
        if it % 25 == 0 or it == 99:
            ex = coracle.reduce_exact("D L2 *", [yh, x, z], [alpha], np.float64, threads=THREADS,
                                      assign_sig="L0 S0 L1 * +")
            r = rs[it].item()
            assert abs(float(r) - ex) <= 1e-12 * abs(ex), (it, float(r), ex)
        coracle.assign("L0 S0 L1 * +", yh, [yh, x], [alpha], threads=THREADS)
    assert Y.to_array().tobytes() == yh.tobytes()


def test_sharded_reduction_partials_combine_like_ranks():
    """Emulate G ranks on one GPU: each block's partial via SALT_PARTIAL, then
    salt_reduce_finish over the G partials (the all-gathered layout) —
    within tolerance of exact and deterministic."""
    n = (1 << 26) + 12345
    x, X = host_and_dev(3, 5, n, np.float64)
    y, Y = host_and_dev(3, 6, n, np.float64)
    ex = coracle.reduce_exact("L0 L1 *", [x, y], [], np.float64, threads=THREADS)
    lib = _native.lib()
    ws = torch.zeros(lib.salt_reduce_workspace_bytes(), dtype=torch.uint8, device="cuda")
    stream = torch.cuda.current_stream().cuda_stream
    for G in (1, 2, 4, 8):
        parts = torch.empty(2 * G, dtype=torch.float64, device="cuda")
        for r in range(G):
            lo, hi = shard_bounds(n, G, r)
            leaves, keep = _native.ptr_array([X.tensor[lo:hi].data_ptr(), Y.tensor[lo:hi].data_ptr()])
            sc, keep2 = _native.double_array([])
            _native.check(lib.salt_reduce(1, b"L0 L1 *", leaves, 2, sc, 0, hi - lo, _native.SALT_PARTIAL,
                                          ws.data_ptr(), ws.numel(), parts[2 * r:].data_ptr(), None, stream))
        out = torch.empty(1, dtype=torch.float64, device="cuda")
        _native.check(lib.salt_reduce_finish(1, parts.data_ptr(), G, 0, out.data_ptr(), None, stream))
        got = out.item()
        assert abs(got - ex) <= 1e-12 * abs(ex), (G, got, ex)


def test_sharded_vector_world1_through_public_api():
    n = 100_001
    x = synth.block(3, 7, 0, n, np.float64)
    y = synth.block(3, 8, 0, n, np.float64)
    X = lv.ShardedVector.from_global(x, "f64", device="cuda")
    Y = lv.ShardedVector.from_global(y, "f64", device="cuda")
    Z = lv.ShardedVector.zeros(n, "f64", device="cuda")
    Z.assign(2.0 * X - Y)
    assert same_bits(Z.to_array(), restate.eval_sig("S0 L0 * L1 -", [x, y], [2.0], "f64"))
    r = lv.dot(X, Y)
    ex = restate.exact_sum(x * y)
    assert abs(float(r) - ex) <= 1e-12 * abs(ex)
    assert lv.norm2(X) == np.sqrt(np.float64(lv.dot(X, X)))


def _torchrun_dist_check(exchange):
    import json
    import socket
    import subprocess
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parents[1]
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ngpu = torch.cuda.device_count()
    env = {**os.environ, "SALT_EXCHANGE": exchange}
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        f"--nproc-per-node={ngpu}", "--master-addr", "127.0.0.1", "--master-port",
                        str(port), str(root / "tools" / "dist_check.py")],
                       capture_output=True, text=True, timeout=600, cwd=root, env=env)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
    line = [ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1]
    res = json.loads(line)
    assert res["ok"] and res["world"] == ngpu, res
    return res


def test_sharded_path_under_torchrun_peer_and_nccl_agree():
    """tools/dist_check.py under torchrun (one process per visible GPU; one
    here), once with the in-kernel NVLink peer exchange and once with the
    NCCL all-gather fallback: both pass the oracle checks and give the same
    bits."""
    peer = _torchrun_dist_check("peer")
    nccl = _torchrun_dist_check("nccl")
    # dot, norm2, axpy_dot, the two lazy dots of the CG step, the fused CG update
    assert peer["peer_exchange_active"] and peer["peer_epochs"] == 6
    assert not nccl["peer_exchange_active"]
    assert peer["values"] == nccl["values"]


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_exchange_protocol_emulated_on_one_gpu(world):
    """The NVLink exchange protocol (publish to every peer, release flag,
    acquire-wait all flags, fold in rank order; epoch-parity double
    buffering) with `world` ranks played by the blocks of ONE cooperative
    launch, over 64 consecutive epochs: every rank gets the same bits, equal
    to the rank-order fold salt_reduce_finish computes."""
    lib = _native.lib()
    rounds = 64
    g = np.random.default_rng(world)
    hi = g.standard_normal((rounds, world)) * 1e3
    lo = hi * 1e-17 * g.standard_normal((rounds, world))
    totals = torch.tensor(np.stack([hi, lo], axis=-1).reshape(-1), dtype=torch.float64, device="cuda")
    results = torch.zeros(rounds * world * 2, dtype=torch.float64, device="cuda")
    scratch = torch.zeros(world * _native.XCHG_BUFFER_BYTES, dtype=torch.uint8, device="cuda")
    stream = torch.cuda.current_stream().cuda_stream
    _native.check(lib.salt_exchange_emulate(world, rounds, 1, totals.data_ptr(), results.data_ptr(),
                                            scratch.data_ptr(), stream))
    res = results.view(rounds, world, 2).cpu().numpy()
    out = torch.empty(1, dtype=torch.float64, device="cuda")
    for r in range(rounds):
        assert all(res[r, k].tobytes() == res[r, 0].tobytes() for k in range(world)), r
        _native.check(lib.salt_reduce_finish(1, totals[r * world * 2:].data_ptr(), world, 0,
                                             out.data_ptr(), None, stream))
        assert np.float64(res[r, 0, 0] + res[r, 0, 1]) == out.item(), r


def test_config5_full_length_on_one_gpu_int64_indexing():
    """Config 5's full global length (2^31 + 5 f64 elements, > INT32_MAX) on
    ONE B200 (3 x 16 GiB resident): the fused axpy->dot step indexes with
    64-bit offsets; y bit-exact and r within 1e-12 of the exact value."""
    n = (1 << 31) + 5
    g = torch.Generator(device="cuda").manual_seed(1109)
    X, Y, Z = (lv.DenseVector.from_tensor(torch.randn(n, dtype=torch.float64, device="cuda", generator=g))
               for _ in range(3))
    x, y, z = (v.to_array() for v in (X, Y, Z))
    alpha = -0.4375
    r = lv.axpy_dot(alpha, X, Y, Z)
    ex = coracle.reduce_exact("D L2 *", [y, x, z], [alpha], np.float64, threads=THREADS,
                              assign_sig="L0 S0 L1 * +")
    assert abs(float(r) - ex) <= 1e-12 * abs(ex), (float(r), ex)
    coracle.assign("L0 S0 L1 * +", y, [y, x], [alpha], threads=THREADS)
    got = Y.to_array()
    assert got.tobytes() == y.tobytes()
    # the last elements (beyond 2^31) were written
    assert got[-1] == y[-1] and got[(1 << 31) + 1] == y[(1 << 31) + 1]
