#!/usr/bin/env python
"""Randomised parity at scale — a long GPU run, not collected by pytest
(test infrastructure, so it may use oracle/ as the checker): seeded
random expression trees at up to 2^26 elements, each evaluated through the
public API on the compiled path (table or NVRTC JIT) and on the interpreter
fallback, compared bit for bit with the NumPy restatement of the
reference's node semantics; reductions of the same trees against the exact
(binary128) sum within the BASELINE tolerance, and compiled == interpreter.

    python tests/stress_parity.py [--trees 60] [--max-logn 26] [--out profiles/r01_parity_stress.json]
"""

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import paper_1109_1264_b200 as lv  # noqa: E402
from oracle import coracle, restate  # noqa: E402  (checker)
from paper_1109_1264_b200 import _native  # noqa: E402
from paper_1109_1264_b200.engine import execute_reduce  # noqa: E402
from paper_1109_1264_b200.expressions import SumNode, as_node, lower  # noqa: E402
from test_gpu_random_trees import random_tree  # noqa: E402

NP = {"f32": np.float32, "f64": np.float64}
TOL = {"f32": 1e-5, "f64": 1e-12}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--trees", type=int, default=60)
    ap.add_argument("--max-logn", type=int, default=26)
    ap.add_argument("--seed", type=int, default=1109)
    ap.add_argument("--out", default=None)
    ap.add_argument("--misalign", action="store_true",
                    help="every operand and the destination is a view at a random element offset (0-8) "
                         "of its own buffer: mostly mixed misalignments (the V = 1 kernels), sometimes "
                         "a shared one (scalar head + 256-bit body)")
    a = ap.parse_args()
    import torch
    lib = _native.lib()
    rng = np.random.default_rng(a.seed)
    rows, fails = [], 0
    t0 = time.time()
    for case in range(a.trees):
        dt = "f32" if case % 2 else "f64"
        logn = int(rng.integers(10, a.max_logn + 1))
        n = (1 << logn) + int(rng.integers(0, 64))
        nv = int(rng.integers(1, 9))
        host = [rng.uniform(-2, 2, n).astype(NP[dt]) for _ in range(nv)]
        if a.misalign:
            share = int(rng.integers(0, 4)) == 0  # a quarter of the cases: one common offset
            offs = [int(rng.integers(0, 9))] * (nv + 1) if share else [int(rng.integers(0, 9)) for _ in range(nv + 1)]
            bufs = [torch.zeros(n + 16, dtype=torch.float32 if dt == "f32" else torch.float64, device="cuda")
                    for _ in range(nv + 1)]
            vecs = []
            for h, b, o in zip(host, bufs, offs):
                b[o:o + n].copy_(torch.from_numpy(h))
                vecs.append(lv.DenseVector.from_tensor(b[o:o + n]))
        else:
            vecs = [lv.DenseVector.from_values(h, dt) for h in host]
        expr = as_node(random_tree(rng, vecs, int(rng.integers(1, 7))))
        lw = lower(expr)
        sig = " ".join(lw.tokens)
        idx = [next(i for i, v in enumerate(vecs) if v is u) for u in lw.vectors]
        leaves = [host[i] for i in idx]
        want = restate.eval_sig(sig, leaves, lw.scalars, dt)
        if a.misalign:
            out = lv.DenseVector.from_tensor(bufs[nv][offs[nv]:offs[nv] + n])
        else:
            out = lv.DenseVector.zeros(n, dt)
        res = {}
        for mode in ("compiled", "interp"):
            lib.salt_set_force_interp(1 if mode == "interp" else 0)
            lib.salt_jit_wait()
            out.assign(expr)
            got = out.to_array()
            res[mode + "_bits"] = bool(np.array_equal(got.view(np.uint8), want.view(np.uint8)) or
                                       np.array_equal(got, want, equal_nan=True))
            res[mode + "_sum"] = float(execute_reduce(SumNode(expr)))
        lib.salt_set_force_interp(0)
        exact = float(coracle.reduce_exact(sig, leaves, lw.scalars, NP[dt], threads=16))
        scale = float(restate.exact_sum(np.abs(want.astype(np.float64)))) if n <= (1 << 22) else abs(exact)
        ok_sum = (not np.isfinite(exact)) or exact == 0 or \
            abs(res["compiled_sum"] - exact) <= TOL[dt] * max(abs(exact), 1e-3 * scale)
        same = res["compiled_sum"] == res["interp_sum"] or (np.isnan(res["compiled_sum"]) and np.isnan(res["interp_sum"]))
        ok = res["compiled_bits"] and res["interp_bits"] and ok_sum and same
        fails += not ok
        rows.append({"case": case, "dtype": dt, "n": n, "sig": sig, "leaves": len(leaves),
                     "elementwise_bit_exact": res["compiled_bits"], "interp_bit_exact": res["interp_bits"],
                     "sum_within_tol": bool(ok_sum), "interp_sum_same_bits": bool(same)})
        print(json.dumps(rows[-1]), flush=True)
    summary = {"trees": a.trees, "failures": fails, "max_logn": a.max_logn, "seed": a.seed,
               "misalign": bool(a.misalign),
               "seconds": round(time.time() - t0, 1), "gpu": __import__("torch").cuda.get_device_name()}
    print(json.dumps(summary))
    if a.out:
        Path(a.out).write_text(json.dumps({"summary": summary, "rows": rows}, indent=1))
    return 1 if fails else 0


if __name__ == "__main__":
    sys.exit(main())
