#!/usr/bin/env python
"""Interpreter kernel vs compiled kernels: device time per launch for the
BASELINE trees at full size (best of 10 after a GPU sleep, CUDA events).

    python tools/interp_probe.py [--n 268435456]
"""

import argparse
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1109_1264_b200 as lv  # noqa: E402
from paper_1109_1264_b200 import _native  # noqa: E402


def best(fn, reps=10):
    for _ in range(3):
        fn()
    t = []
    for _ in range(reps):
        torch.cuda._sleep(100_000)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        t.append(a.elapsed_time(b) * 1e-3)
    return min(t)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1 << 28)
    n = ap.parse_args().n
    v = [lv.DenseVector.from_tensor(torch.rand(n, dtype=torch.float64, device="cuda")) for _ in range(5)]
    cases = {
        "t2": (lambda: v[3].assign(1.25 * v[0] + -0.75 * (v[1] - v[2])), 32),
        "etree_f64": (lambda: v[4].assign(1.25 * (v[0] + v[1]) - 0.75 * (v[2] - v[3]) + 0.5 * v[0]), 40),
        "dot": (lambda: lv.dot(v[0], v[1], lazy=True), 16),
        "axpy_dot": (lambda: lv.axpy_dot(0.5, v[0], v[1], v[2], lazy=True), 32),
    }
    lib = _native.lib()
    out = {"n": n, "gpu": torch.cuda.get_device_name(), "unit": "GB/s (algorithmic bytes / best launch time)"}
    for name, (fn, bpe) in cases.items():
        row = {}
        for mode in (0, 1):
            lib.salt_set_force_interp(mode)
            row["interp" if mode else "compiled"] = round(bpe * n / best(fn) / 1e9, 1)
        lib.salt_set_force_interp(0)
        out[name] = row
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
