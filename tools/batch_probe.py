#!/usr/bin/env python
"""Batched assignments vs one launch per tree: m independent axpys of n
elements (f64), device time (events, host work hidden behind a GPU sleep)
and wall time (host included, expressions prebuilt), best of 5.

    python tools/batch_probe.py
"""

import os
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
from paper_1109_1264_b200.expressions import as_node  # noqa: E402


def device_us(fn):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda._sleep(20_000_000)
    e0.record()
    fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) * 1e3


def wall_us(fn):
    torch.cuda.synchronize()
    t = time.perf_counter()
    fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) * 1e6


def main():
    rows = []
    g = np.random.default_rng(0)
    for n in (1024, 4096, 65536):
        for m in (16, 64, 256, 1024):
            X = [lv.DenseVector.from_values(g.uniform(-1, 1, n), "f64") for _ in range(m)]
            Y = [lv.DenseVector.from_values(g.uniform(-1, 1, n), "f64") for _ in range(m)]
            sts = [(y, as_node(y) + 0.5 * x) for x, y in zip(X, Y)]
            batch = lambda: lv.assign_batch(sts)  # noqa: E731
            loop = lambda: [y.assign(e) for y, e in sts]  # noqa: E731
            batch(), loop()
            r = {"n": n, "m": m,
                 "batch_device_us": round(min(device_us(batch) for _ in range(5)), 1),
                 "loop_device_us": round(min(device_us(loop) for _ in range(5)), 1),
                 "batch_wall_us": round(min(wall_us(batch) for _ in range(5)), 1),
                 "loop_wall_us": round(min(wall_us(loop) for _ in range(5)), 1)}
            rows.append(r)
            print(json.dumps(r), flush=True)
    for n in (1024, 4096):
        for m in (16, 256, 1024):
            P = [tuple(lv.DenseVector.from_values(g.uniform(-1, 1, n), "f64") for _ in range(2))
                 for _ in range(m)]
            batch = lambda: lv.dot_batch(P)  # noqa: E731   one launch per 96 + ONE copy back
            loop = lambda: [lv.dot(x, y) for x, y in P]  # noqa: E731   a sync per dot
            batch(), loop()
            r = {"op": "dot", "n": n, "m": m,
                 "batch_wall_us": round(min(wall_us(batch) for _ in range(5)), 1),
                 "loop_wall_us": round(min(wall_us(loop) for _ in range(5)), 1)}
            rows.append(r)
            print(json.dumps(r), flush=True)
    print(json.dumps({"gpu": torch.cuda.get_device_name(), "what": "m axpys of n f64 elements: "
                      "lv.assign_batch vs one assign per tree; m dots: lv.dot_batch vs lv.dot each"}))


if __name__ == "__main__":
    main()
