"""The C host fast path (csrc/fastpath.c) must not leak references: after
thousands of calls through it, every operand's reference count and the
process's resident memory are where they started."""

import gc
import sys

import numpy as np
import pytest

import paper_1109_1264_b200 as lv

pytestmark = pytest.mark.gpu


def _rss_mb():
    with open("/proc/self/statm") as f:
        return int(f.read().split()[1]) * 4096 / 2**20


def test_fast_path_keeps_reference_counts_and_memory_flat():
    n = 4096
    g = np.random.default_rng(3)
    A, B, C, D = (lv.DenseVector.from_values(g.uniform(-1, 1, n), "f64") for _ in range(4))
    al = lv.DeviceScalar.full(0.5, "f64", device="cuda")

    def calls():
        lv.axpy(0.5, A, B)
        D.assign(1.25 * A + -0.5 * (B - C))
        lv.dot(A, B, lazy=True)
        lv.norm2(A)
        lv.axpy_dot(0.25, A, B, C, lazy=True)
        lv.fused((B, B - al * A), (C, C + al * A), C * C, lazy=True)
        D.assign(al * A + B)
        lv.assign_batch([(D, A + C), (B, B * 0.5)])
        lv.dot_batch([(A, B), (C, C)])
        lv.reduce_batch([A - C, B * 2.0], lazy=True)

    for _ in range(2000):  # warm: JIT, workspaces, allocator pools
        calls()
    gc.collect()
    objs = (A, B, C, D, al)
    before = [sys.getrefcount(o) for o in objs]
    for _ in range(2000):
        calls()
    gc.collect()
    rss1 = _rss_mb()
    for _ in range(4000):  # 28,000 more calls: a leak of even 100 bytes per call shows
        calls()
    gc.collect()
    after = [sys.getrefcount(o) for o in objs]
    assert after == before, (before, after)
    assert _rss_mb() - rss1 < 2, (rss1, _rss_mb())
