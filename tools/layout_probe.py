#!/usr/bin/env python
"""Does the relative placement of operand vectors in HBM change the
streaming rate?  Times f64 dot / fused CG update / T2 at 2^28 with the
operands placed (a) as separate torch allocations of exactly 2 GiB,
(b) through DenseVector.empty (2 GiB + 256 B each), (c) inside one buffer
at controlled offsets.

    python tools/layout_probe.py
"""

import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1109_1264_b200 as lv  # noqa: E402


def t(fn, reps=10):
    for _ in range(3):
        fn()
    best = 1e9
    for _ in range(reps):
        torch.cuda._sleep(100_000)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        best = min(best, a.elapsed_time(b) * 1e-3)
    return best


def cases(vs, n):
    a = lv.DeviceScalar.full(1e-3, "f64", device="cuda")
    out = {}
    out["dot"] = 16 * n / t(lambda: lv.dot(vs[0], vs[1], lazy=True)) / 1e9
    out["t2"] = 32 * n / t(lambda: vs[3].assign(1.25 * vs[0] + -0.75 * (vs[1] - vs[2]))) / 1e9
    out["cg"] = 48 * n / t(lambda: lv.fused((vs[0], vs[0] + a * vs[1]), (vs[2], vs[2] - a * vs[3]),
                                           vs[2] * vs[2], lazy=True)) / 1e9
    return {k: round(v, 1) for k, v in out.items()}


def main():
    n = 1 << 28
    res = {}
    # (a) exact 2 GiB torch allocations
    ts = [torch.rand(n, dtype=torch.float64, device="cuda") for _ in range(4)]
    vs = [lv.DenseVector.from_tensor(x) for x in ts]
    res["separate torch allocations"] = cases(vs, n)
    res["addresses_MiB"] = [(x.data_ptr() - ts[0].data_ptr()) / 2**20 for x in ts]
    del vs, ts
    torch.cuda.empty_cache()
    # (b) DenseVector.empty
    vs = [lv.DenseVector.empty(n, "f64", device="cuda") for _ in range(4)]
    for v in vs:
        v.tensor.uniform_()
    res["DenseVector.empty"] = cases(vs, n)
    res["addresses_MiB_b"] = [(v.tensor.data_ptr() - vs[0].tensor.data_ptr()) / 2**20 for v in vs]
    del vs
    torch.cuda.empty_cache()
    # (c) one buffer, vectors at stride n + off elements
    for off in (0, 32, 512, 4096, 1 << 15, 1 << 18, 1 << 20):
        buf = torch.rand(4 * (n + off), dtype=torch.float64, device="cuda")
        vs = [lv.DenseVector.from_tensor(buf[k * (n + off): k * (n + off) + n]) for k in range(4)]
        res[f"one buffer, stride n+{off} elements ({(n + off) * 8 / 2**20:.3f} MiB)"] = cases(vs, n)
        del vs, buf
        torch.cuda.empty_cache()
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
