#!/usr/bin/env python
"""Product reductions (lv.dot / lv.norm2, lazy) across sizes, clean and dirty
L2, one JSON line per (op, dtype, n, l2):

  clean  before every timed launch a 512 MiB READ sweep (L2 full of clean
         lines, tools/midred_probe.cu's "clean")
  dirty  a 512 MiB WRITE (memset-like fill; L2 full of dirty lines that
         must be written back, config_sweep's flush)

Timing: differential, as tools/c3_probe.cu — R x (sweep + launch) minus
R x sweep, between CUDA events, min of 3 trials — so the launch overhead of
an idle GPU is not in the number.  Run twice to compare combines:

    python tools/reduce_sweep.py > a.jsonl
    SALT_COMBINE=ticket python tools/reduce_sweep.py > b.jsonl
"""

import argparse
import json
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1109_1264_b200 as lv  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--lg", default="20,21,22,23,24,25,26,27,28")
    ap.add_argument("--reps", type=int, default=15)
    a = ap.parse_args()
    sweep = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    fsweep = sweep.view(torch.float32)
    flush = {"clean": lambda: fsweep.sum(), "dirty": lambda: sweep.fill_(7)}
    combine = os.environ.get("SALT_COMBINE", "default")
    for dt in (torch.float64, torch.float32):
        for lg in [int(x) for x in a.lg.split(",")]:
            n = 1 << lg
            x = lv.DenseVector.from_tensor(torch.rand(n, dtype=dt, device="cuda") - 0.5)
            y = lv.DenseVector.from_tensor(torch.rand(n, dtype=dt, device="cuda") - 0.5)
            es = x.tensor.element_size()
            for op, fn, nb in (("dot", lambda: lv.dot(x, y, lazy=True), 2 * es * n),
                               ("norm2", lambda: lv.norm2(x, lazy=True), es * n)):
                fn()
                torch.cuda.synchronize()
                for l2, pre in flush.items():
                    best = float("inf")
                    for _ in range(3):
                        e0, e1, e2, e3 = (torch.cuda.Event(enable_timing=True) for _ in range(4))
                        pre(); fn()
                        e0.record()
                        for _ in range(a.reps):
                            pre(); fn()
                        e1.record()
                        e2.record()
                        for _ in range(a.reps):
                            pre()
                        e3.record()
                        e3.synchronize()
                        d = (e0.elapsed_time(e1) - e2.elapsed_time(e3)) * 1e3 / a.reps
                        best = min(best, d)
                    print(json.dumps({"op": op, "dtype": str(dt).split(".")[-1], "lg": lg, "l2": l2,
                                      "combine": combine, "us": round(best, 3),
                                      "gbs": round(nb / best / 1e3, 1)}), flush=True)
            del x, y


if __name__ == "__main__":
    main()
