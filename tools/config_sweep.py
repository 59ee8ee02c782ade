#!/usr/bin/env python
"""Measure every BASELINE.json config on one B200.

For each config: device time per fused launch (CUDA events, best and
median of R), effective GB/s = algorithmic bytes / time, % of the measured
HBM peak, the same tree as torch eager composition (one kernel per node,
temporaries in HBM — the "BLAS composition" baseline), API latency for the
small config, and the CPU time of the reference algorithm (oracle/ C
restatement, all host threads) on a bounded sample.

    python tools/config_sweep.py --out profiles/r01_configs.jsonl

Algorithmic bytes per unit: s * n * (distinct vectors read + written).
"""

import argparse
import json
import os
import statistics
import sys
import time
from pathlib import Path
# steady-state measurements: build out-of-table trees with NVRTC on first use
# instead of running them on the interpreter meanwhile (tiered JIT)
os.environ.setdefault("SALT_JIT_ASYNC", "0")

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import paper_1109_1264_b200 as lv  # noqa: E402
from paper_1109_1264_b200 import synth  # noqa: E402

PEAK = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"] if (
    ROOT / "MEASURED_PEAKS.json").exists() else 6650.0
THREADS = len(os.sched_getaffinity(0))
FLUSH = None


def flush_l2():
    global FLUSH
    if FLUSH is None:
        FLUSH = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    FLUSH.fill_(7)


def dev_time(fn, reps, warmup=3, flush=False, restore=None):
    for _ in range(warmup):
        if restore:
            restore()
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        if restore:
            restore()
        if flush:
            flush_l2()
        # keep the GPU busy while the host enqueues the timed launch, so the
        # events bracket device time only (not Python launch latency)
        torch.cuda._sleep(200_000)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        e.synchronize()
        ts.append(s.elapsed_time(e) / 1e3)
    return min(ts), statistics.median(ts)


def api_latency(fn, reps=200):
    """Host wall time of one public-API call that returns to the caller,
    including its synchronisation (the cost a Python caller sees)."""
    for _ in range(10):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return min(ts), statistics.median(ts)


def cpu_time(sig, leaves, scalars, dt, reduce=False, reps=3):
    from oracle import coracle

    dt = np.dtype(dt)
    if reduce:
        fn = lambda: coracle.reduce(sig, leaves, scalars, dt, 4, 64 // dt.itemsize, threads=THREADS)
    else:
        out = np.empty(leaves[0].shape[0], dtype=dt)
        fn = lambda: coracle.assign(sig, out, leaves, scalars, threads=THREADS)
    fn()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return min(ts)


def vec(cfg, op, n, dt, lo=0):
    v = lv.DenseVector.empty(n, np.dtype(dt), device="cuda")
    synth.fill_device(v.tensor, cfg, op, lo)
    return v


def rec(out, **kw):
    line = json.dumps(kw)
    print(line, flush=True)
    out.write(line + "\n")
    out.flush()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="profiles/configs.jsonl")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--only", default="1,2,3,4,5", help="comma list of configs to run")
    a = ap.parse_args()
    out = open(a.out, "w")
    R = a.reps
    gpu = torch.cuda.get_device_name()

    only = {int(c) for c in a.only.split(",")}
    if 1 in only:
        c1(out, R, gpu)
    if 2 in only:
        c2(out, R, gpu, a.quick)
    if 3 in only:
        c3(out, R, gpu)
    if 4 in only:
        c4(out, R, gpu)
    if 5 in only:
        c5(out, gpu)
    out.close()


def c1(out, R, gpu):
    # ---------------- C1: daxpy f64 2^20 (L2-resident: 24 MiB) ----------------
    n = 1 << 20
    x, y = vec(1, 0, n, np.float64), vec(1, 1, n, np.float64)
    (al,) = synth.scalars(1, 1)
    y0 = y.tensor.clone()
    restore = lambda: y.tensor.copy_(y0)
    f = lambda: lv.axpy(al, x, y)
    b = 24.0 * n
    hot = dev_time(f, R * 5, restore=restore)
    cold = dev_time(f, R * 5, flush=True, restore=restore)
    lat = api_latency(f)
    tx, ty = x.tensor, y.tensor
    tal = torch.tensor(al, dtype=torch.float64).item()
    tf = lambda: ty.copy_(torch.add(ty, torch.mul(tx, tal)))
    th = dev_time(tf, R * 5, restore=restore)
    hx, hy = synth.block(1, 0, 0, n, np.float64), synth.block(1, 1, 0, n, np.float64)
    ct = cpu_time("L0 S0 L1 * +", [hy, hx], [al], np.float64)
    rec(out, config=1, op="daxpy", dtype="f64", n=n, bytes=b,
        l2_hot_s=hot[0], l2_hot_gbs=b / hot[0] / 1e9, l2_flushed_s=cold[0], l2_flushed_gbs=b / cold[0] / 1e9,
        api_call_s=lat[0], api_call_median_s=lat[1], torch_composed_s=th[0],
        cpu_ref_s=ct, cpu_ref_gbs=b / ct / 1e9, cpu_threads=THREADS, gpu=gpu)
    del x, y, y0


def c2(out, R, gpu, quick):
    # ---------------- C2: a + (b - c) and alpha*a + beta*(b - c), f64 sweep ----------------
    al, be = synth.scalars(2, 2)
    sizes = [1 << p for p in range(10, 29, 2)]
    if quick:
        sizes = [1 << 20, 1 << 28]
    for n in sizes:
        A, B, C = (vec(2, k, n, np.float64) for k in range(3))
        D = lv.DenseVector.empty(n, "f64", device="cuda")
        ta, tb, tc, td = A.tensor, B.tensor, C.tensor, D.tensor
        b = 32.0 * n
        for tree, fn, tfn in (
            ("t1", lambda: D.assign(A + (B - C)), lambda: td.copy_(torch.add(ta, torch.sub(tb, tc)))),
            ("t2", lambda: D.assign(al * A + be * (B - C)),
             lambda: td.copy_(torch.add(torch.mul(ta, al), torch.mul(torch.sub(tb, tc), be)))),
        ):
            flush = n * 32 < (256 << 20)
            g = dev_time(fn, R, flush=flush)
            t = dev_time(tfn, R, flush=flush)
            entry = dict(config=2, op=tree, dtype="f64", n=n, bytes=b, l2_flushed=flush,
                         best_s=g[0], median_s=g[1], gbs=b / g[0] / 1e9, pct_hbm=b / g[0] / 1e9 / PEAK,
                         torch_composed_s=t[0], fusion_speedup=t[0] / g[0], gpu=gpu)
            if n in (1 << 20, 1 << 24):
                hs = [synth.block(2, k, 0, n, np.float64) for k in range(3)]
                sig = "L0 L1 L2 - +" if tree == "t1" else "S0 L0 * S1 L1 L2 - * +"
                ct = cpu_time(sig, hs, [] if tree == "t1" else [al, be], np.float64)
                entry.update(cpu_ref_s=ct, cpu_ref_gbs=b / ct / 1e9, cpu_threads=THREADS)
            if n <= (1 << 16):
                entry["api_call_s"] = api_latency(fn)[0]
            rec(out, **entry)
        del A, B, C, D, ta, tb, tc, td


def c3(out, R, gpu):
    # ---------------- C3: dot / nrm2, f32 + f64, 2^24 and 2^28 ----------------
    for dt in (np.float32, np.float64):
        for n in (1 << 24, 1 << 28):
            X, Y = vec(3, 0, n, dt), vec(3, 1, n, dt)
            s = np.dtype(dt).itemsize
            for op, fn, tfn, nb in (
                ("dot", lambda: lv.dot(X, Y, lazy=True), lambda: torch.dot(X.tensor, Y.tensor), 2 * s * n),
                ("nrm2", lambda: lv.norm2(X, lazy=True), lambda: torch.linalg.vector_norm(X.tensor), s * n),
            ):
                g = dev_time(fn, R)
                t = dev_time(tfn, R)
                entry = dict(config=3, op=op, dtype="f32" if dt == np.float32 else "f64", n=n, bytes=nb,
                             best_s=g[0], median_s=g[1], gbs=nb / g[0] / 1e9, pct_hbm=nb / g[0] / 1e9 / PEAK,
                             torch_library_s=t[0], gpu=gpu)
                if n == 1 << 24:
                    hs = [synth.block(3, k, 0, n, dt) for k in range(2)]
                    sig = "L0 L1 *" if op == "dot" else "L0 L0 *"
                    ct = cpu_time(sig, hs[: 2 if op == "dot" else 1], [], dt, reduce=True)
                    entry.update(cpu_ref_s=ct, cpu_ref_gbs=nb / ct / 1e9, cpu_threads=THREADS)
                rec(out, **entry)
            del X, Y


def c4(out, R, gpu):
    # ---------------- C4: e-tree f32, global 2^30; per-GPU block at G = 1,2,4,8 ----------------
    al, be, ga = synth.scalars(4, 3)
    N = 1 << 30
    ops = [vec(4, k, N, np.float32) for k in range(4)]
    E = lv.DenseVector.empty(N, "f32", device="cuda")
    for G in (1, 2, 4, 8):
        n = N // G
        v = [lv.DenseVector.from_tensor(o.tensor[:n]) for o in ops]
        e = lv.DenseVector.from_tensor(E.tensor[:n])
        fn = lambda: e.assign(al * (v[0] + v[1]) - be * (v[2] - v[3]) + ga * v[0])
        g = dev_time(fn, R)
        b = 20.0 * n
        rec(out, config=4, op="etree", dtype="f32", G=G, n_per_gpu=n, bytes_per_gpu=b, best_s=g[0],
            median_s=g[1], gbs_per_gpu=b / g[0] / 1e9, pct_hbm=b / g[0] / 1e9 / PEAK,
            projected_global_gbs=G * b / g[0] / 1e9, gpu=gpu,
            note="one GPU's block of the G-way partition; no communication (weak per-GPU timing)")
    hs = [synth.block(4, k, 0, 1 << 24, np.float32) for k in range(4)]
    ct = cpu_time("S0 L0 L1 + * S1 L2 L3 - * - S2 L0 * +", hs, [al, be, ga], np.float32)
    rec(out, config=4, op="etree-cpu", dtype="f32", n=1 << 24, cpu_ref_s=ct, cpu_ref_gbs=20.0 * (1 << 24) / ct / 1e9,
        cpu_threads=THREADS)
    del ops, E, v, e


def c5(out, gpu):
    # ---------------- C5: axpy -> dot, f64, 2^28 per GPU (2^31 / 8), 100 iterations ----------------
    n = 1 << 28
    X, Y, Z = (vec(5, k, n, np.float64) for k in range(3))
    (al,) = synth.scalars(5, 1)
    y0 = Y.tensor.clone()
    torch.cuda.synchronize()
    for mode in ("fused", "two-pass"):
        Y.tensor.copy_(y0)
        if mode == "fused":
            step = lambda: lv.axpy_dot(al, X, Y, Z, lazy=True)
        else:
            def step():
                lv.axpy(al, X, Y)
                return lv.dot(Y, Z, lazy=True)
        for _ in range(3):
            step()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        rs = [step() for _ in range(100)]
        e.record()
        e.synchronize()
        el = s.elapsed_time(e) / 1e3
        b = 32.0 * n
        rec(out, config=5, op=f"axpy_dot-{mode}", dtype="f64", n_per_gpu=n, iterations=100, total_s=el,
            per_step_s=el / 100, gbs=b * 100 / el / 1e9, pct_hbm=b * 100 / el / 1e9 / PEAK,
            r_last=float(rs[-1].item()), gpu=gpu,
            note="credited bytes 4*8*n per step (fused compulsory traffic)")
    # a whole CG update (x += a p; r -= a q; rr = r.r) fused vs three passes
    P = Z
    Q = lv.DenseVector.empty(n, "f64", device="cuda")
    Q.tensor.copy_(X.tensor)
    R = Y
    for mode in ("fused", "three-pass"):
        if mode == "fused":
            step = lambda: lv.fused((X, X + al * P), (R, R - al * Q), R * R, lazy=True)
        else:
            def step():
                lv.axpy(al, P, X)
                R.assign(R - al * Q)
                return lv.dot(R, R, lazy=True)
        for _ in range(3):
            step()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(20):
            step()
        e.record()
        e.synchronize()
        el = s.elapsed_time(e) / 1e3 / 20
        b = 48.0 * n  # 4 reads + 2 writes, fused compulsory traffic
        rec(out, config=5, op=f"cg_update-{mode}", dtype="f64", n_per_gpu=n, per_step_s=el,
            gbs=b / el / 1e9, pct_hbm=b / el / 1e9 / PEAK, gpu=gpu,
            note="x += a p; r -= a q; rr = r.r; credited bytes 6*8*n per step")


if __name__ == "__main__":
    main()
