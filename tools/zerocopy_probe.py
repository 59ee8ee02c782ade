#!/usr/bin/env python
"""End-to-end (host vectors) probe: the staged copy pipeline (salt_assign_host,
the product's route) vs ONE fused kernel reading and writing the pinned host
vectors directly over PCIe (zero-copy through UVA: salt_assign on the pinned
pointers).  Same tree and bytes as bench.py's e2e leg (config 2, T2 f64).

    python tools/zerocopy_probe.py [--logn 28] [--reps 5]
"""
import argparse
import ctypes
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_1109_1264_b200 as lv  # noqa: E402
from paper_1109_1264_b200 import _native  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--logn", type=int, default=28)
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    n = 1 << args.logn
    dev = torch.device("cuda:0")
    torch.cuda.set_device(dev)
    g = torch.Generator(device="cpu").manual_seed(3)
    hv = []
    for _ in range(3):
        h = lv.DenseVector.empty(n, "f64", device="cpu")
        src = torch.empty(n, dtype=torch.float64, device=dev).uniform_(-1, 1)
        h.tensor.copy_(src)
        hv.append(h)
        del src
    hd = lv.DenseVector.empty(n, "f64", device="cpu")
    hz = lv.DenseVector.empty(n, "f64", device="cpu")
    ha, hb, hc = hv
    al, be = 1.25, -0.75
    out = {"n": n, "bytes_per_step": 32 * n}

    def staged():
        hd.assign(al * ha + be * (hb - hc))

    lib = _native.lib()
    leaves, _keep_l = _native.ptr_array([t.tensor.data_ptr() for t in hv])
    scal, _keep_s = _native.double_array([al, be])
    stream = torch.cuda.current_stream(dev).cuda_stream

    def zero_copy():
        rc = lib.salt_assign(1, b"S0 L0 * S1 L1 L2 - * +", ctypes.c_void_p(hz.tensor.data_ptr()), leaves, 3,
                             scal, 2, n, ctypes.c_void_p(stream))
        _native.check(rc)
        torch.cuda.synchronize(dev)

    for name, fn in (("staged", staged), ("zero_copy", zero_copy)):
        fn()
        ts = []
        for _ in range(args.reps):
            torch.cuda.synchronize(dev)
            s = time.perf_counter()
            fn()
            torch.cuda.synchronize(dev)
            ts.append(time.perf_counter() - s)
        out[name] = {"best_ms": round(min(ts) * 1e3, 3), "median_ms": round(float(np.median(ts)) * 1e3, 3),
                     "GB/s_best": round(32 * n / min(ts) / 1e9, 2),
                     "GB/s_median": round(32 * n / float(np.median(ts)) / 1e9, 2)}
    out["same_bits"] = bool(torch.equal(hd.tensor.view(torch.int64), hz.tensor.view(torch.int64)))
    print(json.dumps(out))


if __name__ == "__main__":
    main()
