#!/usr/bin/env python
"""BASELINE config 5 in one process over every visible GPU (DeviceGroup):
y = y + alpha*x ; r = dot(y, z), float64, x/y/z block-sharded, 100
iterations, each one fused kernel per device + one NCCL all-reduce of the
per-device partials (salt_allreduce_sum).

    python examples/c5_devicegroup.py [--n 2147483648] [--iters 100] [--check]

--n is the GLOBAL length (default 2^31 on 8 GPUs, i.e. 2^28 per GPU; on
fewer GPUs the default keeps 2^28 per GPU).  --check first compares three
sharded steps at a small length with the same steps on one device.  Device
time is the max over devices between a barrier of events.
"""

import os
import argparse
import json
import sys
from pathlib import Path
# steady-state measurements: build out-of-table trees with NVRTC on first use
# instead of running them on the interpreter meanwhile (tiered JIT)
os.environ.setdefault("SALT_JIT_ASYNC", "0")

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1109_1264_b200 as lv  # noqa: E402
from paper_1109_1264_b200 import synth  # noqa: E402


def check(dg):
    """The sharded step against the same step on one device through the
    public API (lv.axpy_dot): y bit for bit, the dot within 1e-12."""
    n = 1_000_003
    g = np.random.default_rng(5)
    x, y, z = (g.standard_normal(n) for _ in range(3))
    xs, ys, zs = dg.scatter(x, "f64"), dg.scatter(y, "f64"), dg.scatter(z, "f64")
    X, Y, Z = (lv.DenseVector.from_values(v, "f64", device=torch.device("cuda", dg.devices[0]))
               for v in (x, y, z))
    for _ in range(3):
        r = dg.axpy_dot(0.375, xs, ys, zs)
        q = lv.axpy_dot(0.375, X, Y, Z)
        assert dg.gather(ys).tobytes() == Y.to_array().tobytes()
        assert abs(float(r) - float(q)) <= 1e-12 * abs(float(q)), (float(r), float(q))
    return True


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=0)
    ap.add_argument("--iters", type=int, default=100)
    ap.add_argument("--check", action="store_true")
    a = ap.parse_args()
    G = torch.cuda.device_count()
    n = a.n or (1 << 28) * G
    with lv.DeviceGroup(list(range(G))) as dg:
        checked = check(dg) if a.check else None
        xs, ys, zs = (dg.zeros(n, "f64") for _ in range(3))
        for blocks, op in ((xs, 0), (ys, 1), (zs, 2)):
            for (lo, _), b in zip(dg.bounds(n), blocks):
                synth.fill_device(b.tensor, 5, op, lo=lo)
        alpha = synth.scalars(5, 1)[0]
        for _ in range(3):
            dg.axpy_dot(alpha, xs, ys, zs, lazy=True)
        for d in dg.devices:
            torch.cuda.synchronize(d)
        ev = {d: [torch.cuda.Event(enable_timing=True) for _ in range(2)] for d in dg.devices}
        for d in dg.devices:
            with torch.cuda.device(d):
                ev[d][0].record()
        for _ in range(a.iters):
            r = dg.axpy_dot(alpha, xs, ys, zs, lazy=True)
        for d in dg.devices:
            with torch.cuda.device(d):
                ev[d][1].record()
        for d in dg.devices:
            torch.cuda.synchronize(d)
        ms = max(ev[d][0].elapsed_time(ev[d][1]) for d in dg.devices)
        total = r[0].item()
    step_bytes = 32.0 * n  # x, y, z read + y written
    print(json.dumps({"config": 5, "gpus": G, "n_global": n, "iters": a.iters,
                      "ms_per_step": round(ms / a.iters, 4),
                      "GBps_total": round(step_bytes * a.iters / (ms / 1e3) / 1e9, 1),
                      "GBps_per_gpu": round(step_bytes * a.iters / (ms / 1e3) / 1e9 / G, 1),
                      "r_last": total, "checked": checked}))


if __name__ == "__main__":
    main()
