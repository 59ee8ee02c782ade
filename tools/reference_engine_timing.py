#!/usr/bin/env python
"""CPU timings of the reference's hot path on this host, for context beside
the GPU numbers (SURVEY.md §8(d) CPU timing protocol):

  lanevec        the unmodified reference engine (block executor, default
                 plan), imported from baseline/_ref (pip --target install of
                 /root/reference, git-ignored), pinned to one core
  numpy-1core    the whole-array NumPy restatement (oracle/restate.py;
                 bit-identical to the engine), one core
  c-port-1t      the C restatement (oracle/salt_oracle.c), one thread
  c-port-all     the C restatement, all host threads (bench.py's baseline)

GB/s = element size x n x (distinct vectors read + written) / best time.

    python tools/reference_engine_timing.py --out profiles/r01_cpu_reference_engines.json
"""

import argparse
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
REF = ROOT / "baseline" / "_ref"

from oracle import coracle, restate  # noqa: E402

CASES = [
    # name, postfix signature, dtype, n, vectors (distinct reads + write), scalars, kind
    ("daxpy (C1)", "L0 S0 L1 * +", "f64", 1 << 20, 3, [1.25], "assign"),
    ("a+(b-c) (C2 T1)", "L0 L1 L2 - +", "f64", 1 << 20, 4, [], "assign"),
    ("al*a+be*(b-c) (C2 T2)", "S0 L0 * S1 L1 L2 - * +", "f64", 1 << 20, 4, [1.25, -0.5], "assign"),
    ("ddot (C3)", "L0 L1 *", "f64", 1 << 22, 2, [], "reduce"),
    ("sdot (C3)", "L0 L1 *", "f32", 1 << 22, 2, [], "reduce"),
    ("e-tree f32 (C4)", "S0 L0 L1 + * S1 L2 L3 - * - S2 L0 * +", "f32", 1 << 20, 5, [1.25, -0.5, 0.75],
     "assign"),
]


def best(fn, reps):
    fn()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return min(ts)


def lanevec_call(lv, sig, dt, arrays, scalars, kind):
    vecs = [lv.DenseVector.from_values(a, dt) for a in arrays]
    nl = len(arrays)
    if sig == "L0 S0 L1 * +":
        return lambda: lv.axpy(scalars[0], vecs[1], vecs[0])
    if kind == "reduce":
        return lambda: lv.dot(vecs[0], vecs[1])
    d = lv.DenseVector.zeros(len(arrays[0]), dt)
    v = vecs
    if sig == "L0 L1 L2 - +":
        return lambda: d.assign(v[0] + (v[1] - v[2]))
    if sig == "S0 L0 * S1 L1 L2 - * +":
        return lambda: d.assign(scalars[0] * v[0] + scalars[1] * (v[1] - v[2]))
    if nl == 4:
        return lambda: d.assign(scalars[0] * (v[0] + v[1]) - scalars[1] * (v[2] - v[3]) + scalars[2] * v[0])
    raise ValueError(sig)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    threads = len(os.sched_getaffinity(0))
    res = {"host_threads": threads, "cases": []}
    lv = None
    if REF.exists():
        sys.path.insert(0, str(REF))
        import lanevec as lv  # noqa: F811
    g = np.random.default_rng(7)
    all_cpus = os.sched_getaffinity(0)
    for name, sig, dt, n, nvec, scalars, kind in CASES:
        npdt = np.float32 if dt == "f32" else np.float64
        nl = max(int(t[1:]) for t in sig.split() if t[0] == "L") + 1
        arrays = [g.uniform(-1, 1, n).astype(npdt) for _ in range(nl)]
        nbytes = np.dtype(npdt).itemsize * n * nvec
        row = {"case": name, "dtype": dt, "n": n, "bytes": nbytes}
        os.sched_setaffinity(0, {min(all_cpus)})  # one core
        if lv is not None:
            t = best(lanevec_call(lv, sig, dt, arrays, scalars, kind), 2)
            row["lanevec_1core_gbs"] = nbytes / t / 1e9
        if kind == "assign":
            t = best(lambda: restate.eval_sig(sig, arrays, scalars, dt), 5)
        else:
            t = best(lambda: restate.engine_reduce(restate.eval_sig(sig, arrays, [], dt), 4, 64 // np.dtype(npdt).itemsize), 5)
        row["numpy_1core_gbs"] = nbytes / t / 1e9
        out = np.empty(n, dtype=npdt)
        if kind == "assign":
            c1 = lambda: coracle.assign(sig, out, arrays, scalars, threads=1)
            ca = lambda: coracle.assign(sig, out, arrays, scalars, threads=threads)
        else:
            c1 = lambda: coracle.reduce(sig, arrays, [], dt, 4, 64 // np.dtype(npdt).itemsize, threads=1)
            ca = lambda: coracle.reduce(sig, arrays, [], dt, 4, 64 // np.dtype(npdt).itemsize, threads=threads)
        row["c_port_1thread_gbs"] = nbytes / best(c1, 5) / 1e9
        os.sched_setaffinity(0, all_cpus)
        row["c_port_all_threads_gbs"] = nbytes / best(ca, 5) / 1e9
        res["cases"].append(row)
        print(json.dumps(row), flush=True)
    res["lanevec_available"] = lv is not None
    if a.out:
        Path(a.out).write_text(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
