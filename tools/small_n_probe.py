#!/usr/bin/env python
"""Device time per launch for mid-size (L2-resident) vectors: 200 back-to-back
launches between two events (no host gaps: the GPU queue stays full), per
size.  Used with SALT_ASSIGN_TILES / SALT_REDUCE_TILES to tune the work per
CTA at sizes where launch and ramp costs matter."""

import os
import json
import sys
from pathlib import Path
# steady-state measurements: build out-of-table trees with NVRTC on first use
# instead of running them on the interpreter meanwhile (tiered JIT)
os.environ.setdefault("SALT_JIT_ASYNC", "0")

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1109_1264_b200 as lv  # noqa: E402


def main():
    import argparse

    ap = argparse.ArgumentParser()
    ap.add_argument("--logn", default="12,16,18,20,22,24")
    ap.add_argument("--ops", default="axpy,t2,dot,axpy_dot")
    args = ap.parse_args()
    out = {}
    for logn in map(int, args.logn.split(",")):
        n = 1 << logn
        v = [lv.DenseVector.from_tensor(torch.rand(n, dtype=torch.float64, device="cuda")) for _ in range(4)]
        f = [lv.DenseVector.from_tensor(torch.rand(n, dtype=torch.float32, device="cuda")) for _ in range(2)]
        cases = {
            "axpy": (lambda: lv.axpy(0.5, v[0], v[1]), 24),
            "t2": (lambda: v[3].assign(1.25 * v[0] + -0.5 * (v[1] - v[2])), 32),
            "dot": (lambda: lv.dot(v[0], v[1], lazy=True), 16),
            "nrm2": (lambda: lv.norm2(v[0], lazy=True), 8),
            "sdot": (lambda: lv.dot(f[0], f[1], lazy=True), 8),
            "axpy_dot": (lambda: lv.axpy_dot(0.5, v[0], v[1], v[2], lazy=True), 32),
        }
        cases = {k: c for k, c in cases.items() if k in args.ops.split(",")}
        for name, (fn, bpe) in cases.items():
            for _ in range(20):
                fn()
            torch.cuda.synchronize()
            # capture 200 launches in a graph so host issue cost is excluded
            g = torch.cuda.CUDAGraph()
            s = torch.cuda.Stream()
            s.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s):
                fn()
            torch.cuda.current_stream().wait_stream(s)
            with torch.cuda.graph(g):
                for _ in range(200):
                    fn()
            g.replay()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            g.replay()
            e1.record()
            e1.synchronize()
            us = e0.elapsed_time(e1) * 1e3 / 200
            out[f"{name}@2^{logn}"] = {"us_per_launch": round(us, 3), "GBps": round(bpe * n / us / 1e3, 1)}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
