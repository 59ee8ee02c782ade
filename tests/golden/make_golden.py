"""Generate tests/golden/*.npz from the REFERENCE implementation itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports the unmodified reference package `lanevec` from
/root/reference/pkg/src, evaluates seeded inputs through its public API
(DenseVector.assign, ops.*, execute_reduce, call_trace) and stores inputs and
outputs.  The fixtures travel with the repo; /root/reference does not exist
on the GPU box, so nothing at test time imports the reference.

Fixtures
  elementwise.npz  trees x dtypes x lengths: operands, scalars, reference output
  reductions.npz   dot / sum / norm2 / tree-sums: operands, reference engine
                   value for several plans, exact fsum value
  fused.npz        axpy then dot (config 5 building block): y_out and r
  specials.npz     inf / nan / -0.0 / subnormal operands through the trees
  traces.npz       call_trace event lists for several plans
  special_reductions.npz  sum / dot over operands with inf, -inf, NaN, max
"""

import json
import math
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent
SEED = 20260814  # the reference acceptance suite's seed (test_acceptance.py:30)

sys.path.insert(0, str(REF))
import lanevec as lv  # noqa: E402
from lanevec.engine import call_trace, execute_reduce  # noqa: E402
from lanevec.expressions import AssignNode, ScaleNode, SumNode, as_node  # noqa: E402
from lanevec.lanes import scalar_backend, wide_backend  # noqa: E402

DTYPES = ("f32", "f64")
NP = {"f32": np.float32, "f64": np.float64}
SMALL = [0, 1, 2, 3, 5, 7, 8, 9, 15, 16, 17, 31, 32, 33, 63, 64, 65, 100, 127, 128, 129]
BIG = [1000, 4097]

# name -> (postfix signature, number of operand vectors, number of scalars,
#          builder(vectors, scalars, dest) -> evaluates through the reference API)
TREES = {
    "copy": ("L0", 1, 0, lambda v, s, d: d.assign(v[0])),
    "scaled_copy": ("S0 L0 *", 1, 1, lambda v, s, d: lv.scaled_copy(s[0], v[0], d)),
    "t1": ("L0 L1 L2 - +", 3, 0, lambda v, s, d: d.assign(v[0] + (v[1] - v[2]))),
    "t2": ("S0 L0 * S1 L1 L2 - * +", 3, 2,
           lambda v, s, d: d.assign(s[0] * v[0] + s[1] * (v[1] - v[2]))),
    "etree": ("S0 L0 L1 + * S1 L2 L3 - * - S2 L0 * +", 4, 3,
              lambda v, s, d: d.assign(s[0] * (v[0] + v[1]) - s[1] * (v[2] - v[3]) + s[2] * v[0])),
    "mul3": ("L0 L1 * L2 *", 3, 0, lambda v, s, d: d.assign(v[0] * v[1] * v[2])),
    "neg_sum": ("S0 L0 L1 + *", 2, 1, lambda v, s, d: d.assign(-(v[0] + v[1]))),
    "mixed": ("L0 L1 * L2 L0 * - S0 L1 * +", 3, 1,
              lambda v, s, d: d.assign((v[0] * v[1] - v[2] * v[0]) + s[0] * v[1])),
    "scale_right": ("S0 L0 L1 - *", 2, 1, lambda v, s, d: d.assign((v[0] - v[1]) * s[0])),
}
# In-place ops: (signature with L0 = destination, builder)
INPLACE = {
    "scal": ("S0 L0 *", 1, 1, lambda v, s: lv.scal(s[0], v[0])),
    "axpy": ("L0 S0 L1 * +", 2, 1, lambda v, s: lv.axpy(s[0], v[1], v[0])),
}


def rng(*key):
    return np.random.default_rng([SEED, *key])


def gen_elementwise():
    out = {}
    meta = []
    for ti, (name, (sig, nv, ns, build)) in enumerate(TREES.items()):
        lengths = SMALL + (BIG if name in ("t1", "t2", "etree", "scaled_copy") else [])
        for di, dt in enumerate(DTYPES):
            for n in lengths:
                g = rng(1, ti, di, n)
                vals = [g.uniform(-1, 1, n).astype(NP[dt]) for _ in range(nv)]
                scal = [float(x) for x in g.uniform(-2, 2, ns)]
                if name == "neg_sum":
                    scal = [-1.0]  # unary minus is ScaleNode(-1, ...) (expressions.py:99-100)
                vecs = [lv.DenseVector.from_values(a, dt) for a in vals]
                d = lv.DenseVector.zeros(n, dt)
                build(vecs, scal, d)
                key = f"{name}|{dt}|{n}"
                for k, a in enumerate(vals):
                    out[f"{key}|in{k}"] = a
                out[f"{key}|sc"] = np.array(scal, dtype=np.float64)
                out[f"{key}|out"] = d.to_array()
                meta.append([name, sig, dt, n, nv, ns])
    for ti, (name, (sig, nv, ns, build)) in enumerate(INPLACE.items()):
        for di, dt in enumerate(DTYPES):
            for n in SMALL + BIG:
                g = rng(2, ti, di, n)
                vals = [g.uniform(-1, 1, n).astype(NP[dt]) for _ in range(nv)]
                scal = [float(x) for x in g.uniform(-2, 2, ns)]
                vecs = [lv.DenseVector.from_values(a, dt) for a in vals]
                build(vecs, scal)
                key = f"{name}|{dt}|{n}"
                for k, a in enumerate(vals):
                    out[f"{key}|in{k}"] = a
                out[f"{key}|sc"] = np.array(scal, dtype=np.float64)
                out[f"{key}|out"] = vecs[0].to_array()
                meta.append([name, sig, dt, n, nv, ns])
    out["meta"] = np.array(json.dumps(meta))
    np.savez_compressed(OUT / "elementwise.npz", **out)
    return len(meta)


RED_TREES = {
    "dot": ("L0 L1 *", 2, lambda v, o: lv.dot(v[0], v[1], **o)),
    "sum": ("L0", 1, lambda v, o: lv.sum(v[0], **o)),
    "norm2": ("L0 L0 *", 1, lambda v, o: lv.norm2(v[0], **o)),
    "sum_t1": ("L0 L1 L2 - +", 3,
               lambda v, o: execute_reduce(SumNode(as_node(v[0]) + (as_node(v[1]) - as_node(v[2]))), **o)),
}
PLANS = {"default": {}, "u1": {"unroll": 1}, "u8": {"unroll": 8}, "scalar": "scalar"}


def gen_reductions():
    out = {}
    meta = []
    for ti, (name, (sig, nv, build)) in enumerate(RED_TREES.items()):
        for di, dt in enumerate(DTYPES):
            for n in SMALL + BIG:
                for dist in ("pos", "normal"):
                    g = rng(3, ti, di, n, 0 if dist == "pos" else 1)
                    if dist == "pos":
                        vals = [g.uniform(0.25, 1.25, n).astype(NP[dt]) for _ in range(nv)]
                    else:
                        vals = [g.standard_normal(n).astype(NP[dt]) for _ in range(nv)]
                    vecs = [lv.DenseVector.from_values(a, dt) for a in vals]
                    key = f"{name}|{dt}|{n}|{dist}"
                    for k, a in enumerate(vals):
                        out[f"{key}|in{k}"] = a
                    for pname, opts in PLANS.items():
                        if opts == "scalar":
                            opts = {"backend": scalar_backend(dt)}
                        r = build(vecs, opts)
                        out[f"{key}|ref_{pname}"] = np.array([r], dtype=NP[dt])
                    # exact oracle of the reference's acceptance test (:95-100)
                    x = vals[0]
                    if name == "dot":
                        terms = (vals[0] * vals[1]).astype(np.float64)
                    elif name == "norm2":
                        terms = (x * x).astype(np.float64)
                    elif name == "sum":
                        terms = x.astype(np.float64)
                    else:
                        terms = (vals[0] + (vals[1] - vals[2])).astype(np.float64)
                    exact = math.fsum(terms.tolist())
                    if name == "norm2":
                        exact = math.sqrt(exact)
                    out[f"{key}|exact"] = np.array([exact])
                    meta.append([name, sig, dt, n, dist, nv])
    out["meta"] = np.array(json.dumps(meta))
    np.savez_compressed(OUT / "reductions.npz", **out)
    return len(meta)


def gen_fused():
    """Config 5's step: y = y + alpha*x (axpy), then r = dot(y, z)."""
    out = {}
    meta = []
    for di, dt in enumerate(DTYPES):
        for n in SMALL + BIG:
            g = rng(4, di, n)
            x, y, z = (g.standard_normal(n).astype(NP[dt]) for _ in range(3))
            alpha = float(g.uniform(-1, 1))
            X, Y, Z = (lv.DenseVector.from_values(a, dt) for a in (x, y, z))
            lv.axpy(alpha, X, Y)
            r = lv.dot(Y, Z)
            key = f"{dt}|{n}"
            out[f"{key}|x"], out[f"{key}|y"], out[f"{key}|z"] = x, y, z
            out[f"{key}|alpha"] = np.array([alpha])
            out[f"{key}|y_out"] = Y.to_array()
            out[f"{key}|r_ref"] = np.array([r], dtype=NP[dt])
            out[f"{key}|r_exact"] = np.array([math.fsum((Y.to_array() * z).astype(np.float64).tolist())])
            meta.append([dt, n])
    out["meta"] = np.array(json.dumps(meta))
    np.savez_compressed(OUT / "fused.npz", **out)
    return len(meta)


def gen_specials():
    out = {}
    meta = []
    for dt in DTYPES:
        tiny = np.finfo(NP[dt]).tiny
        special = np.array([0.0, -0.0, np.inf, -np.inf, np.nan, 1.0, -1.0, tiny, tiny / 8,
                            -tiny / 1024, np.finfo(NP[dt]).max, -np.finfo(NP[dt]).max, 1e-310 if dt == "f64" else 1e-40,
                            3.0, 0.5, 2.0 ** -20], dtype=NP[dt])
        k = special.shape[0]
        a = np.repeat(special, k)
        b = np.tile(special, k)
        c = np.roll(b, 3)
        for name in ("t1", "t2", "mul3", "etree"):
            sig, nv, ns, build = TREES[name]
            vals = [a, b, c, np.roll(a, 5)][:nv]
            scal = [1.5, -0.75, 2.0 ** -30][:ns]
            vecs = [lv.DenseVector.from_values(v, dt) for v in vals]
            d = lv.DenseVector.zeros(a.shape[0], dt)
            with np.errstate(all="ignore"):
                build(vecs, scal, d)
            key = f"{name}|{dt}"
            for i, v in enumerate(vals):
                out[f"{key}|in{i}"] = v
            out[f"{key}|sc"] = np.array(scal)
            out[f"{key}|out"] = d.to_array()
            meta.append([name, sig, dt, int(a.shape[0]), nv, ns])
    out["meta"] = np.array(json.dumps(meta))
    np.savez_compressed(OUT / "specials.npz", **out)
    return len(meta)


def gen_special_reductions():
    """Reductions over operands holding inf / -inf / NaN / huge values."""
    out = {}
    meta = []
    cases = {
        "inf": lambda x: np.concatenate([x, [np.inf]]),
        "ninf": lambda x: np.concatenate([[-np.inf], x]),
        "both_inf": lambda x: np.concatenate([[np.inf], x, [-np.inf]]),
        "nan": lambda x: np.concatenate([x[:10], [np.nan], x[10:]]),
        "huge": lambda x: np.concatenate([x, [np.finfo(x.dtype).max] * 3]),
    }
    for dt in DTYPES:
        base = rng(5, 0 if dt == "f32" else 1).uniform(-1, 1, 997).astype(NP[dt])
        for cname, mk in cases.items():
            x = mk(base).astype(NP[dt])
            X = lv.DenseVector.from_values(x, dt)
            with np.errstate(all="ignore"):
                r_sum = lv.sum(X)
                r_dot = lv.dot(X, X)
            key = f"{cname}|{dt}"
            out[f"{key}|x"] = x
            out[f"{key}|sum"] = np.array([r_sum], dtype=NP[dt])
            out[f"{key}|dot"] = np.array([r_dot], dtype=NP[dt])
            meta.append([cname, dt, int(x.shape[0])])
    out["meta"] = np.array(json.dumps(meta))
    np.savez_compressed(OUT / "special_reductions.npz", **out)
    return len(meta)


def gen_traces():
    out = {}
    meta = []
    cases = [
        ("assign_scale", 16, "f32", 4, 2, 1),
        ("assign_scale", 37, "f32", 4, 4, 2),
        ("assign_axpy", 103, "f32", 4, 8, 4),
        ("assign_axpy", 103, "f64", 8, 2, 1),
        ("reduce_dot", 20, "f32", 4, 2, 1),
        ("reduce_dot", 0, "f32", 4, 4, 1),
        ("assign_scale", 9, "f32", 1, 1, 1),
        ("assign_axpy", 130, "f64", 8, None, None),
    ]
    for ci, (kind, n, dt, width, unroll, packages) in enumerate(cases):
        x = lv.DenseVector.from_values(np.arange(n), dt)
        y = lv.DenseVector.from_values(np.arange(n)[::-1].copy(), dt)
        if kind == "assign_scale":
            root = AssignNode(as_node(y), ScaleNode(2.0, as_node(x)))
        elif kind == "assign_axpy":
            root = AssignNode(as_node(y), as_node(y) + ScaleNode(0.5, as_node(x)))
        else:
            root = SumNode(as_node(x) * as_node(y))
        backend = scalar_backend(dt) if width == 1 else wide_backend(dt, width)
        opts = {"backend": backend}
        if unroll is not None:
            opts["unroll"] = unroll
        if packages is not None:
            opts["packages"] = packages
        tr = call_trace(root, **opts)
        enc = [[e.kind, -1 if e.index is None else e.index, -1 if e.slot is None else e.slot] for e in tr]
        out[f"case{ci}"] = np.array(json.dumps(enc))
        meta.append([kind, n, dt, width, unroll, packages])
    out["meta"] = np.array(json.dumps(meta))
    np.savez_compressed(OUT / "traces.npz", **out)
    return len(meta)


if __name__ == "__main__":
    print("elementwise cases:", gen_elementwise())
    print("reduction cases:", gen_reductions())
    print("fused cases:", gen_fused())
    print("special cases:", gen_specials())
    print("trace cases:", gen_traces())
    print("special reduction cases:", gen_special_reductions())
