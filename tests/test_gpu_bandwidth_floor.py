"""Bandwidth floors for the hot kernels (a regression guard, not a
benchmark): each must stream at >= 85 % of what it measured on a B200 in
round 1 (profiles/r01_launch_bounds.txt, profiles/r01_configs.jsonl).  A
codegen regression — e.g. ptxas spending more registers and losing
occupancy — shows up here as a failure instead of silently in bench.py."""

import pytest
import torch

import paper_1109_1264_b200 as lv

pytestmark = pytest.mark.gpu

N = 1 << 27
FLOOR = 0.85
MEASURED = {  # GB/s at 2^28 on one B200 (round 1)
    "t2": 7300, "dot64": 7330, "nrm2_32": 6800, "axpy_dot": 7250, "cg_update_device_scalar": 7120,
}


def best_time(fn, reps=10):
    for _ in range(3):
        fn()
    lv.jit_wait()  # out-of-table trees (device-scalar CG update): time the compiled kernel
    best = float("inf")
    for _ in range(reps):
        torch.cuda._sleep(100_000)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        best = min(best, a.elapsed_time(b) * 1e-3)
    return best


def test_hot_kernels_stream_near_their_measured_rate():
    v = [lv.DenseVector.from_tensor(torch.rand(N, dtype=torch.float64, device="cuda")) for _ in range(4)]
    f = lv.DenseVector.from_tensor(torch.rand(2 * N, dtype=torch.float32, device="cuda"))
    a = lv.DeviceScalar.full(1e-3, "f64", device="cuda")
    cases = {
        "t2": (lambda: v[3].assign(1.25 * v[0] + -0.5 * (v[1] - v[2])), 32 * N),
        "dot64": (lambda: lv.dot(v[0], v[1], lazy=True), 16 * N),
        "nrm2_32": (lambda: lv.norm2(f, lazy=True), 8 * N),
        "axpy_dot": (lambda: lv.axpy_dot(0.5, v[0], v[1], v[2], lazy=True), 32 * N),
        "cg_update_device_scalar": (lambda: lv.fused((v[0], v[0] + a * v[1]), (v[2], v[2] - a * v[3]),
                                                     v[2] * v[2], lazy=True), 48 * N),
    }
    got = {k: nbytes / best_time(fn) / 1e9 for k, (fn, nbytes) in cases.items()}
    low = {k: round(g) for k, g in got.items() if g < FLOOR * MEASURED[k]}
    assert not low, f"below {FLOOR:.0%} of the round-1 rate: {low} (all: {got})"
