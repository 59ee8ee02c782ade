#!/usr/bin/env python
"""Mid sizes (2^22-2^27 elements; 32 MB-1 GB per vector, around the 126 MB
L2): why a single reduction launch there runs below the streaming rate.

For each size and op, device time per launch measured three ways:
  single      one launch after a 100 us GPU sleep (config_sweep's method)
  b2b         20 back-to-back launches between two events, averaged
  b2b_clean   same, but each launch preceded by a 512 MiB READ sweep that
              leaves the L2 full of clean lines (no inputs resident)
  diff        R x (read sweep + launch) minus R x (read sweep), per launch:
              the clean-L2 cost without the ~2 us tick of the event clock
  diff_dirty  the same with a 512 MiB fill (L2 full of dirty lines, the
              flush config_sweep and the driver's rules use)
and the same for the torch library call (torch.dot / vector_norm / eager T1).

    python tools/mid_size_probe.py [--out profiles/r01_mid_sizes.json]
"""

import os
import argparse
import json
import sys
from pathlib import Path
# steady-state measurements: build out-of-table trees with NVRTC on first use
# instead of running them on the interpreter meanwhile (tiered JIT)
os.environ.setdefault("SALT_JIT_ASYNC", "0")

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1109_1264_b200 as lv  # noqa: E402

SINK = None


def clean_l2():
    global SINK
    if SINK is None:
        SINK = torch.ones(64 << 20, dtype=torch.float64, device="cuda")
    SINK.sum()


def single(fn, reps=10):
    ts = []
    for _ in range(reps):
        torch.cuda._sleep(200_000)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    return min(ts)


def b2b(fn, reps=20, clean=False):
    best = float("inf")
    for _ in range(3):
        if clean:
            evs = []
            for _ in range(reps):
                clean_l2()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                fn()
                b.record()
                evs.append((a, b))
            torch.cuda.synchronize()
            best = min(best, min(a.elapsed_time(b) for a, b in evs) * 1e3)
        else:
            torch.cuda._sleep(100_000)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(reps):
                fn()
            b.record()
            b.synchronize()
            best = min(best, a.elapsed_time(b) * 1e3 / reps)
    return best


DIRTY = None


def dirty_l2():
    global DIRTY
    if DIRTY is None:
        DIRTY = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    DIRTY.fill_(7)


def diff(fn, reps=40, dirty=False):
    sweep = dirty_l2 if dirty else clean_l2
    best = float("inf")
    for _ in range(3):
        a, b, c = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        sweep()
        fn()
        a.record()
        for _ in range(reps):
            sweep()
            fn()
        b.record()
        for _ in range(reps):
            sweep()
        c.record()
        c.synchronize()
        best = min(best, (a.elapsed_time(b) - b.elapsed_time(c)) * 1e3 / reps)
    return best


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--logn", default="22,23,24,25,26,27")
    ap.add_argument("--ops", default="nrm2,dot,t1")
    ap.add_argument("--dtypes", default="f64,f32")
    ap.add_argument("--modes", default="single,b2b,b2b_clean")
    ap.add_argument("--no-torch", action="store_true")
    args = ap.parse_args()
    res = {"gpu": torch.cuda.get_device_name(), "unit": "us per launch", "rows": []}
    for logn in map(int, args.logn.split(",")):
        n = 1 << logn
        for dt, tdt in (("f64", torch.float64), ("f32", torch.float32)):
            if dt not in args.dtypes.split(","):
                continue
            v = [lv.DenseVector.from_tensor(torch.rand(n, dtype=tdt, device="cuda")) for _ in range(4)]
            t = [x.tensor for x in v]
            s = t[0].element_size()
            cases = {
                "nrm2": (lambda: lv.norm2(v[0], lazy=True), lambda: torch.linalg.vector_norm(t[0]), s),
                "dot": (lambda: lv.dot(v[0], v[1], lazy=True), lambda: torch.dot(t[0], t[1]), 2 * s),
                "t1": (lambda: v[3].assign(v[0] + (v[1] - v[2])),
                       lambda: torch.add(t[0], torch.sub(t[1], t[2]), out=t[3]), 4 * s),
            }
            for op, (fn, tfn, bpe) in cases.items():
                if op not in args.ops.split(","):
                    continue
                for _ in range(5):
                    fn()
                    tfn()
                row = {"op": op, "dtype": dt, "n": n, "MB": round(bpe * n / 1e6, 1)}
                for name, f in (("salt", fn), ("torch", tfn))[: 1 if args.no_torch else 2]:
                    for mode, m in (("single", lambda f=f: single(f)), ("b2b", lambda f=f: b2b(f)),
                                    ("b2b_clean", lambda f=f: b2b(f, clean=True)),
                                    ("diff", lambda f=f: diff(f)), ("diff_dirty", lambda f=f: diff(f, dirty=True))):
                        if mode not in args.modes.split(","):
                            continue
                        us = m()
                        row[f"{name}_{mode}_us"] = round(us, 2)
                        row[f"{name}_{mode}_GBps"] = round(bpe * n / us / 1e3, 1)
                res["rows"].append(row)
                print(json.dumps(row), flush=True)
            del v, t
    if args.out:
        Path(args.out).write_text(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
