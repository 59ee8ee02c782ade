"""NumPy restatement of the reference's evaluation (TEST INFRASTRUCTURE ONLY).

Every function cites the reference code it restates
(/root/reference/pkg/src/lanevec/...).  Arrays in, arrays/scalars out; no
dependency on the product package.
"""

import math

import numpy as np

__all__ = [
    "DTYPES",
    "eval_sig",
    "default_plan",
    "footprint_of",
    "engine_reduce",
    "engine_reduce_loop",
    "exact_sum",
    "exact_reduce",
    "oracle_dot",
    "oracle_sum",
    "oracle_scal",
    "oracle_axpy",
    "oracle_scaled_copy",
    "kahan_sum",
    "SIGS",
]

DTYPES = {"f32": np.dtype(np.float32), "f64": np.dtype(np.float64)}

# Canonical postfix signatures of the trees the reference's ops and the
# BASELINE configs build (leaves numbered by first appearance, scalars by
# appearance; a ScaleNode puts alpha LEFT of its child, expressions.py:320).
SIGS = {
    "copy": "L0",
    "scale": "S0 L0 *",  # scal (dest aliases L0) / scaled_copy (ops.py:23-45)
    "axpy": "L0 S0 L1 * +",  # y + alpha*x with L0 = y = dest (ops.py:32-36)
    "t1": "L0 L1 L2 - +",  # d = a + (b - c)
    "t2": "S0 L0 * S1 L1 L2 - * +",  # d = alpha*a + beta*(b - c)
    "etree": "S0 L0 L1 + * S1 L2 L3 - * - S2 L0 * +",  # alpha(a+b) - beta(c-d) + gamma*a
    "sum": "L0",
    "dot": "L0 L1 *",
    "sq": "L0 L0 *",
}


def eval_sig(sig: str, leaves, scalars, dtype) -> np.ndarray:
    """Evaluate a postfix tree over whole arrays in the element type.

    One NumPy ufunc per node, left operand first: the same IEEE operation per
    element as _BinaryNode.block_op (expressions.py:248-249, operator
    add/sub/mul :255-270) and ScaleNode.block_op (alpha * block, :319-320),
    so the result is bit-identical to the reference engine for every plan
    (the engine only changes how elements are grouped, not the per-element
    arithmetic).
    """
    dt = DTYPES[dtype] if isinstance(dtype, str) else np.dtype(dtype)
    leaves = [np.asarray(v, dtype=dt) for v in leaves]
    sc = [dt.type(s) for s in scalars]
    st = []
    for tok in sig.split():
        if tok[0] == "L":
            st.append(leaves[int(tok[1:])])
        elif tok[0] == "S":
            st.append(sc[int(tok[1:])])
        else:
            b = st.pop()
            a = st.pop()
            with np.errstate(all="ignore"):
                if tok == "+":
                    r = np.add(a, b, dtype=dt)
                elif tok == "-":
                    r = np.subtract(a, b, dtype=dt)
                elif tok == "*":
                    r = np.multiply(a, b, dtype=dt)
                else:
                    raise ValueError(f"bad token {tok!r}")
            st.append(r)
    if len(st) != 1:
        raise ValueError(f"malformed signature {sig!r}")
    out = st[0]
    n = len(leaves[0]) if leaves else 0
    return np.broadcast_to(np.asarray(out, dtype=dt), (n,)).copy()


def footprint_of(sig: str, root: str) -> int:
    """Register footprint of the tree (expressions.py:159-161, :205-207,
    :284-286, :350-354, :418-420): 1 per leaf occurrence and per scale node,
    +1 for an Assign or Sum root.  In postfix every scalar marks one
    ScaleNode."""
    toks = sig.split()
    fp = sum(1 for t in toks if t[0] in "LS")
    return fp + (1 if root in ("assign", "sum") else 0)


def default_plan(footprint: int, dtype) -> tuple:
    """(U, W) of select_plan with the default wide backend (engine.py:103-145,
    lanes.py:178-190): W fills 64 bytes; U = largest of 1,2,4,8 with
    U*footprint <= 16."""
    w = 64 // (DTYPES[dtype] if isinstance(dtype, str) else np.dtype(dtype)).itemsize
    fit = [u for u in (1, 2, 4, 8) if u * footprint <= 16]
    return (max(fit) if fit else 1), w


def engine_reduce_loop(values: np.ndarray, unroll: int, width: int):
    """_run_block_reduce (engine.py:267-292) literally: flat accumulator of
    B = U*W lanes, `acc += block` per iteration, scalar remainder, then
    combine_partials (expressions.py:470-480).  O(n/B) Python iterations."""
    dt = values.dtype
    b = unroll * width
    nm = values.shape[0] & ~(b - 1)
    acc = np.zeros(b, dtype=dt)
    for i in range(0, nm, b):
        acc += values[i : i + b]
    rem = dt.type(0)
    for v in values[nm:]:
        rem = rem + v
    return _combine(acc, unroll, width, rem, nm > 0)


def engine_reduce(values: np.ndarray, unroll: int, width: int):
    """Same result as engine_reduce_loop, vectorised with np.add.accumulate
    down the rows of the (n/B, B) view: accumulate is strictly sequential, so
    each lane j is summed ((acc_j + r0_j) + r1_j) + ... in row order, exactly
    the per-lane order of `acc += block` (np.add.reduce is NOT used: for
    B == 1 it would switch to pairwise summation).  Pinned against the loop
    form and the golden vectors in tests."""
    dt = values.dtype
    b = unroll * width
    nm = values.shape[0] & ~(b - 1)
    acc = np.zeros(b, dtype=dt)
    rows = values[:nm].reshape(-1, b)
    step = max(1, (1 << 20) // b)
    for r in range(0, rows.shape[0], step):
        block = np.concatenate([acc[None, :], rows[r : r + step]], axis=0)
        acc = np.add.accumulate(block, axis=0, dtype=dt)[-1].copy()
    rem = dt.type(0)
    for v in values[nm:]:
        rem = rem + v
    return _combine(acc, unroll, width, rem, nm > 0)


def _combine(acc, unroll, width, rem, have_rows):
    # The reference always folds its U rows, which are zero when the main
    # loop did not run (engine.py:291-292), so have_rows needs no branch.
    total = None
    for s in range(unroll):
        row = acc[s * width : (s + 1) * width]
        h = row[0]
        for k in range(1, width):
            h = h + row[k]
        total = h if total is None else total + h
    return total + rem


def exact_sum(values: np.ndarray, chunk: int = 1 << 22) -> float:
    """Sum of element-typed values as math.fsum of their exact f64 images
    (test_acceptance.py:95-100).  Large inputs go chunk by chunk: each
    chunk contributes its correctly rounded sum s and the correctly rounded
    residual fsum(chunk - s), so the result is within a few ulp^2 of exact."""
    v = np.asarray(values).astype(np.float64, copy=False)
    if v.shape[0] <= chunk:
        return math.fsum(v.tolist())
    # fsum of per-chunk fsums has error <= nchunks * ulp/2 of the chunk sums'
    # scale; tighten by carrying each chunk's rounding error explicitly.
    parts = []
    for i in range(0, v.shape[0], chunk):
        c = v[i : i + chunk].tolist()
        s = math.fsum(c)
        parts.append(s)
        parts.append(math.fsum(c + [-s]))  # exact residual of this chunk
    return math.fsum(parts)


def exact_reduce(sig: str, leaves, scalars, dtype) -> float:
    """Acceptance oracle of the reference (test_acceptance.py:95-100): the
    tree's element-typed values summed exactly."""
    return exact_sum(eval_sig(sig, leaves, scalars, dtype))


# ---- the reference's scalar-loop oracles (oracle.py:26-69), restated ----
def oracle_dot(x, y):
    if len(x) != len(y):
        raise ValueError(f"length mismatch: {len(x)} vs {len(y)}")
    acc = 0
    for a, b in zip(x, y):
        acc = acc + a * b
    return acc


def oracle_sum(x):
    acc = 0
    for a in x:
        acc = acc + a
    return acc


def oracle_scal(alpha, x) -> list:
    return [alpha * a for a in x]


def oracle_axpy(alpha, x, y) -> list:
    if len(x) != len(y):
        raise ValueError(f"length mismatch: {len(x)} vs {len(y)}")
    return [b + alpha * a for a, b in zip(x, y)]


def oracle_scaled_copy(alpha, x) -> list:
    return [alpha * a for a in x]


def kahan_sum(values):
    """Neumaier-compensated left-to-right sum in the input's type."""
    total = 0
    comp = 0
    for v in values:
        t = total + v
        if abs(total) >= abs(v):
            comp = comp + ((total - t) + v)
        else:
            comp = comp + ((v - t) + total)
        total = t
    return total + comp
