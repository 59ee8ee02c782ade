"""salt_group_fused (csrc/salt_abi_group.inc): concurrent issue of one tree
on G members from persistent host threads.  With one GPU the members share
device 0 on separate streams; every member's result must carry the bits of
its own serial salt_fused call (assignments bit-exact, reductions the same
partials), and errors come back with the failing member named."""

import ctypes

import numpy as np
import pytest
import torch

import paper_1109_1264_b200 as lv
from oracle import restate
from paper_1109_1264_b200 import _native

pytestmark = pytest.mark.gpu

SIG4 = "S0 L0 L1 + * S1 L2 L3 - * - S2 L0 * +"


def _group(G):
    devs = (ctypes.c_int * G)(*([0] * G))
    g = ctypes.c_void_p()
    _native.check(_native.lib().salt_group_create(G, ctypes.addressof(devs), ctypes.addressof(g)))
    return g


@pytest.mark.parametrize("G", [1, 3, 8])
def test_group_assign_bits_match_oracle(G):
    lib = _native.lib()
    rng = np.random.default_rng([11, G])
    ns = [int(rng.integers(1, 300_000)) for _ in range(G)]
    host = [[rng.uniform(-1, 1, n).astype(np.float32) for _ in range(4)] for n in ns]
    dev = [[torch.from_numpy(h).cuda() for h in hs] for hs in host]
    outs = [torch.empty(n, dtype=torch.float32, device="cuda") for n in ns]
    streams = [torch.cuda.Stream() for _ in range(G)]
    sc = [1.25, -0.5, 0.75]
    grp = _group(G)
    try:
        assert lib.salt_group_size(grp) == G
        dsts, k1 = _native.ptr_array([o.data_ptr() for o in outs])
        leaves, k2 = _native.ptr_array([t.data_ptr() for ts in dev for t in ts])
        scal, k3 = _native.double_array(sc)
        nn, k4 = _native.i64_array(ns)
        strs, k5 = _native.ptr_array([s.cuda_stream for s in streams])
        _native.check(lib.salt_group_fused(grp, _native.SALT_F32, SIG4.encode(), None, dsts, 1, leaves, 4,
                                           scal, 3, None, 0, nn, 0, None, 0, None, strs))
        torch.cuda.synchronize()
        for g in range(G):
            want = restate.eval_sig(SIG4, host[g], sc, "f32")
            assert outs[g].cpu().numpy().tobytes() == want.tobytes()
        st, en = (ctypes.c_int64 * G)(), (ctypes.c_int64 * G)()
        _native.check(lib.salt_group_issue_times(grp, ctypes.addressof(st), ctypes.addressof(en)))
        assert all(0 <= s <= e for s, e in zip(st, en))
    finally:
        _native.check(lib.salt_group_destroy(grp))


def test_group_fused_partials_match_serial():
    """axpy->dot on 4 members: destinations bit-exact and each partial equal
    to the member's own serial SALT_PARTIAL call."""
    lib = _native.lib()
    G, n = 4, 1_000_003
    rng = np.random.default_rng(5)
    xs = [rng.standard_normal(n) for _ in range(G)]
    ys = [rng.standard_normal(n) for _ in range(G)]
    zs = [rng.standard_normal(n) for _ in range(G)]
    X = [torch.from_numpy(v).cuda() for v in xs]
    Y = [torch.from_numpy(v).cuda() for v in ys]
    Y2 = [t.clone() for t in Y]
    Z = [torch.from_numpy(v).cuda() for v in zs]
    streams = [torch.cuda.Stream() for _ in range(G)]
    wsb = lib.salt_reduce_workspace_bytes()
    ws = [torch.zeros(wsb + 256, dtype=torch.uint8, device="cuda") for _ in range(G)]
    parts = [torch.empty(2, dtype=torch.float64, device="cuda") for _ in range(G)]
    E = lv.expressions
    Yv, Xv, Zv = (lv.DenseVector.from_tensor(t) for t in (Y2[0], X[0], Z[0]))
    node = E.FusedNode([E.AssignNode(E.as_node(Yv), E.as_node(Yv) + 0.5 * E.as_node(Xv))],
                       E.SumNode(E.as_node(Yv) * E.as_node(Zv)))
    asig, rsig, lw0, _ = node.lower()  # the lowering lv.axpy_dot uses
    nl = len(lw0.vectors)
    idx = {id(Yv): 0, id(Xv): 1, id(Zv): 2}
    order = lambda g, T: [T[idx[id(v)]][g] for v in lw0.vectors]  # noqa: E731
    grp = _group(G)
    try:
        leaves, k1 = _native.ptr_array([t.data_ptr() for g in range(G) for t in order(g, (Y, X, Z))])
        dsts, k2 = _native.ptr_array([Y[g].data_ptr() for g in range(G)])
        scal, k3 = _native.double_array(list(lw0.scalars))
        nn, k4 = _native.i64_array([n] * G)
        wss, k5 = _native.ptr_array([w.data_ptr() for w in ws])
        outs, k6 = _native.ptr_array([p.data_ptr() for p in parts])
        strs, k7 = _native.ptr_array([s.cuda_stream for s in streams])
        _native.check(lib.salt_group_fused(grp, _native.SALT_F64, asig.encode(), rsig.encode(), dsts, 1,
                                           leaves, nl, scal, len(lw0.scalars), None, 0, nn,
                                           _native.SALT_PARTIAL, wss, wsb, outs, strs))
        torch.cuda.synchronize()
    finally:
        _native.check(lib.salt_group_destroy(grp))
    for g in range(G):
        want_y = restate.eval_sig("L0 S0 L1 * +", [ys[g], xs[g]], [0.5], "f64")
        assert Y[g].cpu().numpy().tobytes() == want_y.tobytes()
        # serial reference partial on a fresh copy
        y2 = torch.from_numpy(ys[g]).cuda()
        p2 = torch.empty(2, dtype=torch.float64, device="cuda")
        w2 = torch.zeros(wsb + 256, dtype=torch.uint8, device="cuda")
        lv_, k8 = _native.ptr_array([t.data_ptr() for t in order(0, ([y2], [X[g]], [Z[g]]))])
        dp, k9 = _native.ptr_array([y2.data_ptr()])
        _native.check(lib.salt_fused(_native.SALT_F64, asig.encode(), rsig.encode(), dp, 1, lv_, nl, scal,
                                     len(lw0.scalars), None, 0, n, _native.SALT_PARTIAL, w2.data_ptr(), wsb,
                                     p2.data_ptr(), None, torch.cuda.current_stream().cuda_stream))
        torch.cuda.synchronize()
        assert torch.equal(p2, parts[g])


def test_group_error_names_the_member():
    lib = _native.lib()
    grp = _group(2)
    try:
        a = torch.zeros(10, dtype=torch.float64, device="cuda")
        dsts, k1 = _native.ptr_array([a.data_ptr(), a.data_ptr()])
        leaves, k2 = _native.ptr_array([a.data_ptr(), 0])  # member 1: NULL leaf
        nn, k3 = _native.i64_array([10, 10])
        strs, k4 = _native.ptr_array([0, 0])
        scal, k5 = _native.double_array([])
        rc = lib.salt_group_fused(grp, _native.SALT_F64, b"L0 L0 +", None, dsts, 1, leaves, 1, scal, 0,
                                  None, 0, nn, 0, None, 0, None, strs)
        assert rc != 0
        assert b"group member 1" in lib.salt_last_error()
    finally:
        _native.check(lib.salt_group_destroy(grp))


def test_devicegroup_assign_and_fused_use_the_group():
    n = 200_001
    rng = np.random.default_rng(9)
    a, b, c, d = (rng.uniform(-1, 1, n) for _ in range(4))
    with lv.DeviceGroup([0]) as dg:
        A, B, C, Dd = (dg.scatter(v, "f32") for v in (a, b, c, d))
        E = dg.zeros(n, "f32")
        dg.assign([(E[g], 1.25 * (A[g] + B[g]) - -0.5 * (C[g] - Dd[g]) + 0.75 * A[g]) for g in range(dg.size)])
        want = restate.eval_sig(SIG4, [v.astype(np.float32) for v in (a, b, c, d)], [1.25, -0.5, 0.75], "f32")
        assert dg.gather(E).tobytes() == want.tobytes()
        st = dg.issue_times()
        assert len(st) == 1 and st[0][0] <= st[0][1]


def _exchange_descs(G, timeout_ns=10_000_000_000):
    """G in-kernel exchange descriptors whose buffers all live on device 0
    (members on one GPU: no peer access needed)."""
    nb = _native.XCHG_BUFFER_BYTES
    bufs = [torch.zeros(nb // 8, dtype=torch.int64, device="cuda") for _ in range(G)]
    errs = [torch.zeros(1, dtype=torch.int32, device="cuda") for _ in range(G)]
    descs = (_native.Exchange * G)()
    for g in range(G):
        d = descs[g]
        d.rank, d.world, d.epoch, d.timeout_ns, d.error = g, G, 1, timeout_ns, errs[g].data_ptr()
        for p in range(G):
            d.slots[p] = bufs[p].data_ptr()
            d.flags[p] = bufs[p].data_ptr() + 2 * _native.XCHG_MAX_RANKS * 16
    return descs, bufs, errs


@pytest.mark.timeout(300)
@pytest.mark.parametrize("G", [2, 4])
def test_group_in_kernel_exchange_between_concurrent_kernels(G):
    """G members on ONE GPU, each a dot over its own block, trading their
    totals inside the reduction kernels (two concurrently running kernels
    waiting on each other's flags): every member ends with the same bits,
    the rank-order fold of the members' partials, for 3 consecutive epochs."""
    lib = _native.lib()
    n = (1 << 22) + 5
    rng = np.random.default_rng([21, G])
    xs = [rng.standard_normal(n) for _ in range(G)]
    ys = [rng.standard_normal(n) for _ in range(G)]
    X = [torch.from_numpy(v).cuda() for v in xs]
    Y = [torch.from_numpy(v).cuda() for v in ys]
    streams = [torch.cuda.Stream() for _ in range(G)]
    wsb = lib.salt_reduce_workspace_bytes()
    ws = [torch.zeros(wsb + 256, dtype=torch.uint8, device="cuda") for _ in range(G)]
    outs = [torch.zeros(2, dtype=torch.float64, device="cuda") for _ in range(G)]
    descs, bufs, errs = _exchange_descs(G)
    grp = _group(G)
    try:
        leaves, k1 = _native.ptr_array([t.data_ptr() for g in range(G) for t in (X[g], Y[g])])
        sc, k2 = _native.double_array([])
        nn, k3 = _native.i64_array([n] * G)
        wss, k4 = _native.ptr_array([w.data_ptr() for w in ws])
        ops, k5 = _native.ptr_array([o.data_ptr() for o in outs])
        strs, k6 = _native.ptr_array([s.cuda_stream for s in streams])
        for epoch in (1, 2, 3):
            for d in descs:
                d.epoch = epoch
            _native.check(lib.salt_group_fused_exchange(grp, _native.SALT_F64, None, b"L0 L1 *", None, 0, leaves,
                                                        2, sc, 0, None, 0, nn, 0, wss, wsb,
                                                        ctypes.addressof(descs), ops, strs))
            torch.cuda.synchronize()
            vals = [o[0].item() for o in outs]
            assert all(np.float64(v).tobytes() == np.float64(vals[0]).tobytes() for v in vals)
            ex = restate.exact_sum(np.concatenate([x * y for x, y in zip(xs, ys)]))
            assert abs(vals[0] - ex) <= 1e-12 * abs(ex)
        assert all(int(e.item()) == 0 for e in errs)
    finally:
        _native.check(lib.salt_group_destroy(grp))


def test_devicegroup_peer_exchange_matches_the_nccl_route():
    n = 300_001
    rng = np.random.default_rng(31)
    x, y, z = (rng.standard_normal(n) for _ in range(3))
    res = {}
    for ex in ("nccl", "peer"):
        with lv.DeviceGroup([0], exchange=ex) as dg:
            X, Y, Z = dg.scatter(x, "f64"), dg.scatter(y, "f64"), dg.scatter(z, "f64")
            res[ex] = (dg.dot(X, Y), dg.norm2(Z), dg.axpy_dot(0.5, X, Y, Z),
                       dg.dot(X, Z, lazy=True)[0].item())
    assert [np.float64(v).tobytes() for v in res["nccl"]] == [np.float64(v).tobytes() for v in res["peer"]]
