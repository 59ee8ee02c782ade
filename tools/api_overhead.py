#!/usr/bin/env python
"""Host-side cost per call of the public API for launch-bound (small) vectors.

Times N back-to-back calls without synchronising in between (so the number
is the host issue cost, the GPU runs behind), for:
  the public API (lv.axpy, d.assign(tree), lv.dot(lazy=True), lv.axpy_dot),
  the bare C-ABI call with prebuilt arguments (ctypes),
  the same trees as torch eager ops,
  and one CUDA-graph replay of 100 captured fused steps.

    python tools/api_overhead.py [--n 1024] [--calls 2000]
"""

import os
import argparse
import json
import sys
import time
from pathlib import Path
# steady-state measurements: build out-of-table trees with NVRTC on first use
# instead of running them on the interpreter meanwhile (tiered JIT)
os.environ.setdefault("SALT_JIT_ASYNC", "0")

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1109_1264_b200 as lv  # noqa: E402
from paper_1109_1264_b200 import _native  # noqa: E402


def per_call(fn, calls):
    for _ in range(50):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(calls):
        fn()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    return (t1 - t0) / calls, (t2 - t0) / calls


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1024)
    ap.add_argument("--calls", type=int, default=2000)
    a = ap.parse_args()
    n = a.n
    g = np.random.default_rng(0)
    x, y, z, w = (lv.DenseVector.from_values(g.uniform(-1, 1, n), "f64", device="cuda") for _ in range(4))
    tx, ty, tz, tw = x.tensor, y.tensor, z.tensor, w.tensor
    lib = _native.lib()
    sig = b"S0 L0 * S1 L1 L2 - * +"
    leaves, keep = _native.ptr_array([tx.data_ptr(), ty.data_ptr(), tz.data_ptr()])
    sc, keep2 = _native.double_array([1.25, -0.5])
    stream = torch.cuda.current_stream().cuda_stream
    res = {"n": n, "gpu": torch.cuda.get_device_name()}
    ds = lv.DeviceScalar.full(0.5, "f64", device="cuda")
    cases = {
        "lv.axpy": lambda: lv.axpy(0.5, x, y),
        "d.assign(alpha*a+beta*(b-c))": lambda: w.assign(1.25 * x + -0.5 * (y - z)),
        "lv.dot(lazy=True)": lambda: lv.dot(x, y, lazy=True),
        "lv.dot (returns host scalar, synchronises)": lambda: lv.dot(x, y),
        "lv.axpy_dot(lazy=True)": lambda: lv.axpy_dot(0.5, x, y, z, lazy=True),
        "lv.fused CG update (host scalar, lazy)": lambda: lv.fused((x, x + 0.5 * y), (z, z - 0.5 * w),
                                                                   z * z, lazy=True),
        "lv.fused CG update (DeviceScalar alpha, lazy)": lambda: lv.fused((x, x + ds * y), (z, z - ds * w),
                                                                          z * z, lazy=True),
        "d.assign(DeviceScalar*a + b)": lambda: w.assign(ds * x + y),
        "C ABI salt_assign (prebuilt args)": lambda: lib.salt_assign(1, sig, tw.data_ptr(), leaves, 3, sc, 2,
                                                                   n, stream),
        "torch eager alpha*a+beta*(b-c)": lambda: tw.copy_(torch.add(torch.mul(tx, 1.25),
                                                                     torch.mul(torch.sub(ty, tz), -0.5))),
        "torch eager dot": lambda: torch.dot(tx, ty),
    }
    for name, fn in cases.items():
        issue, total = per_call(fn, a.calls)
        res[name] = {"issue_us": round(issue * 1e6, 2), "throughput_us": round(total * 1e6, 2)}
    # CUDA graph of 100 fused axpy->dot steps
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        lv.axpy_dot(0.5, x, y, z, lazy=True)
    torch.cuda.current_stream().wait_stream(s)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        for _ in range(100):
            lv.axpy_dot(0.5, x, y, z, lazy=True)
    issue, total = per_call(graph.replay, max(10, a.calls // 100))
    res["cuda graph: 100 x axpy_dot, per step"] = {"issue_us": round(issue * 1e6 / 100, 3),
                                                   "throughput_us": round(total * 1e6 / 100, 3)}
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
