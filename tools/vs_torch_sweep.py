#!/usr/bin/env python
"""Ours vs torch's own kernels, every named op x f32/f64 x 2^10..2^28: device
time per launch of 50 back-to-back launches replayed from a CUDA graph (no
host gaps), best of 5 replays.  Flags every case where torch is more than
3 % faster (profiles/r02_vs_torch.json)."""
import json
import os
import sys
from pathlib import Path

os.environ.setdefault("SALT_JIT_ASYNC", "0")
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1109_1264_b200 as lv  # noqa: E402


def dev_us(fn, reps=50):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
    torch.cuda.current_stream().wait_stream(s)
    with torch.cuda.graph(g):
        for _ in range(reps):
            fn()
    g.replay()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / reps * 1e3)
    return best


def main():
    rows, slower = [], []
    for dt, tdt in (("f64", torch.float64), ("f32", torch.float32)):
        for lg in range(10, 29, 2):
            n = 1 << lg
            ta, tb, tc, td = (torch.rand(n, dtype=tdt, device="cuda") for _ in range(4))
            a, b, c, d = (lv.DenseVector.from_tensor(t) for t in (ta, tb, tc, td))
            tmp = torch.empty_like(ta)
            reps = 50 if lg <= 24 else 10
            cases = {
                "axpy": (lambda: lv.axpy(0.5, a, b), lambda: tb.add_(ta, alpha=0.5)),
                "scal": (lambda: lv.scal(1.0001, a), lambda: ta.mul_(1.0001)),
                "scaled_copy": (lambda: lv.scaled_copy(0.5, a, d), lambda: torch.mul(ta, 0.5, out=td)),
                "t1": (lambda: d.assign(a + (b - c)),
                       lambda: torch.add(ta, torch.sub(tb, tc, out=tmp), out=td)),
                "dot": (lambda: lv.dot(a, b, lazy=True), lambda: torch.dot(ta, tb)),
                "nrm2": (lambda: lv.norm2(a, lazy=True), lambda: torch.linalg.vector_norm(ta)),
                "sum": (lambda: lv.sum(a, lazy=True), lambda: torch.sum(ta)),
            }
            for op, (ours, theirs) in cases.items():
                o, t = dev_us(ours, reps), dev_us(theirs, reps)
                row = {"dtype": dt, "log2n": lg, "op": op, "ours_us": round(o, 3), "torch_us": round(t, 3),
                       "torch_over_ours": round(t / o, 3)}
                rows.append(row)
                if t < 0.97 * o:
                    slower.append(row)
            del a, b, c, d, ta, tb, tc, td, tmp
            torch.cuda.empty_cache()
    print(json.dumps({"gpu": torch.cuda.get_device_name(0), "protocol": __doc__, "rows": rows,
                      "torch_faster_by_3pct": slower}, indent=1))


if __name__ == "__main__":
    main()
