"""Named level-1 operations (reference pkg/src/lanevec/ops.py:18-55).

Same names, arguments, tree shapes and return types.  Each call is one fused
kernel launch.  Two B200 additions:

  * `norm2` finishes with the square root inside the reduction kernel
    (SALT_SQRT) instead of a separate host np.sqrt — same value: the sum is
    rounded to the element type first, then sqrt'ed in the element type,
    exactly as np.sqrt(dot(x, x)) does (ops.py:53-55);
  * `axpy_dot` fuses y = y + alpha*x with dot(y, z) into ONE pass (the
    building block of BASELINE config 5); the reference composes two
    traversals.

Reductions accept `lazy=True` to return a DeviceScalar without a host
synchronisation (for solver loops).
"""

from . import _native
from .engine import execute_assign, execute_assign_reduce, execute_fused, execute_reduce
from .expressions import (
    AssignNode,
    AssignReduceNode,
    FusedNode,
    MulNode,
    ScaleNode,
    SumNode,
    as_node,
)

__all__ = ["dot", "scal", "axpy", "scaled_copy", "sum", "norm2", "axpy_dot", "fused", "assign_batch",
           "reduce_batch", "dot_batch", "norm2_batch", "jit_wait"]


def _op(sig, dest, leaves, alpha=None, flags=0, lazy=False):
    """C fast path for a named operation on plain device vectors (no node
    objects; csrc/fastpath.c `op`): the same signature, scalars and kernel
    as the node path below.  None = not eligible."""
    fast = _native.fastpath()
    if fast is None:
        return None
    return fast.op(sig, dest, leaves, alpha, flags, lazy)


def _lazy_only(options):
    return not options or (len(options) == 1 and "lazy" in options)


def dot(x, y, **options):
    """Sum of elementwise products of two equal-length vectors."""
    if _lazy_only(options):
        r = _op(b"L0 L0 *" if x is y else b"L0 L1 *", None, (x,) if x is y else (x, y),
                lazy=options.get("lazy", False))
        if r is not None:
            return r
    return execute_reduce(SumNode(MulNode(as_node(x), as_node(y))), **options)


def scal(alpha, x, **options) -> None:
    """In-place x = alpha * x (exact aliasing of source and destination)."""
    if not options and _op(b"S0 L0 *", x, (x,), alpha) is not None:
        return
    execute_assign(AssignNode(as_node(x), ScaleNode(alpha, as_node(x))), **options)


def axpy(alpha, x, y, **options) -> None:
    """In-place y = y + alpha * x."""
    if not options and x is not y and _op(b"L0 S0 L1 * +", y, (y, x), alpha) is not None:
        return
    execute_assign(AssignNode(as_node(y), as_node(y) + ScaleNode(alpha, as_node(x))), **options)


def scaled_copy(alpha, x, out, **options) -> None:
    """out = alpha * x in one traversal (n reads + n writes); out must not
    overlap x."""
    if not options and _op(b"S0 L0 *", out, (x,), alpha) is not None:
        return
    execute_assign(AssignNode(as_node(out), ScaleNode(alpha, as_node(x))), **options)


def sum(x, **options):  # noqa: A001 - reference name
    """Sum of all elements."""
    if _lazy_only(options):
        r = _op(b"L0", None, (x,), lazy=options.get("lazy", False))
        if r is not None:
            return r
    return execute_reduce(SumNode(as_node(x)), **options)


def norm2(x, **options):
    """Euclidean norm sqrt(dot(x, x)), no overflow scaling (as the reference)."""
    if _lazy_only(options):
        r = _op(b"L0 L0 *", None, (x,), flags=_native.SALT_SQRT, lazy=options.get("lazy", False))
        if r is not None:
            return r
    return execute_reduce(
        SumNode(MulNode(as_node(x), as_node(x))), _flags=_native.SALT_SQRT, **options
    )


def axpy_dot(alpha, x, y, z, **options):
    """y = y + alpha*x, then return dot(y_new, z) — one fused pass reading
    x, y, z once and writing y once."""
    yl = as_node(y)
    root = AssignReduceNode(
        AssignNode(yl, yl + ScaleNode(alpha, as_node(x))),
        SumNode(MulNode(as_node(y), as_node(z))),
    )
    return execute_assign_reduce(root, **options)


def fused(*statements, lazy=False):
    """Run statements in one pass: `(dest, expression)` pairs for
    assignments, optionally a final bare expression to sum, e.g. a
    conjugate-gradient update

        rr = lv.fused((x, x + a * p), (r, r - a * q), r * r)

    Same results as running them one after another (later statements see
    earlier assignments); returns the sum, or None without one."""
    # common case straight to the C fast path, without node objects (it
    # declines anything unusual; the node path below then validates/raises)
    pairs = statements if statements and isinstance(statements[-1], tuple) else statements[:-1]
    if 1 <= len(pairs) <= _native.SALT_MAX_ROOTS and all(
            isinstance(st, tuple) and len(st) == 2 for st in pairs):
        fast = _native.fastpath()
        if fast is not None:
            total = None if pairs is statements else statements[-1]
            r = fast.fused(pairs, total, 0, lazy)
            if r is not None:
                return r[0]
    assigns, total = [], None
    for k, st in enumerate(statements):
        if isinstance(st, tuple) and len(st) == 2:
            assigns.append(AssignNode(as_node(st[0]), as_node(st[1])))
        elif k == len(statements) - 1:
            total = SumNode(as_node(st))
        else:
            raise TypeError("only the last statement may be a bare expression (the sum)")
    return execute_fused(FusedNode(assigns, total), lazy=lazy)


def assign_batch(statements) -> int:
    """Evaluate many INDEPENDENT assignments `(dest, expression)` at once.
    Statements whose operands are device vectors and share a tree shape and
    element type run as ONE kernel launch per up to 96 of them
    (salt_assign_batch) — for launch-bound sizes, where one launch per tree
    costs more than the work; each result has the bits of its own
    `dest.assign(expression)`.  Every statement is validated like `assign`
    (dtype, lengths) before anything runs.  A destination may alias its own
    statement's operands (as in axpy) but must not be used by any other
    statement of the batch (ValueError): the statements run concurrently.
    Returns how many statements went through a batched launch."""
    statements = list(statements)
    fast = _native.fastpath()
    if fast is not None:
        r = fast.assign_batch(statements)  # C: walk, check, group, launch
        if r is not None:
            return r
    from .engine import _check_assign_batch

    items = _check_assign_batch(statements)
    from .runtime import run_assign_batch

    return run_assign_batch(items)


def jit_wait() -> None:
    """Block until every background NVRTC build has finished (trees outside
    the compiled-in table run on the bit-identical interpreter kernel until
    their build is done).  Call it after warming up, before timing."""
    failed = _native.lib().salt_jit_wait()
    if failed:
        raise RuntimeError(f"{failed} background JIT build(s) failed; those trees stay on the interpreter")


def reduce_batch(expressions, *, sqrt=False, lazy=False) -> list:
    """Sums of many INDEPENDENT expressions (the reduce counterpart of
    assign_batch): small ones (at most two tiles, a few thousand elements)
    sharing a tree shape and element type run as ONE launch per up to 96,
    and all of a group's results return to the host in one copy; each result
    has the bits of its own `execute_reduce(SumNode(expression))` (sqrt=True:
    of `norm2`).  lazy=True returns DeviceScalars."""
    from .engine import _lower_sum
    from .runtime import batch_results, run_reduce_batch

    expressions = list(expressions)
    flags = _native.SALT_SQRT if sqrt else 0
    fast = _native.fastpath()
    if fast is not None and expressions:
        roots = [SumNode(as_node(e)) for e in expressions]  # validates dtypes
        dts = {r.dtype for r in roots}
        if len(dts) == 1:
            r = fast.reduce_batch([root.child for root in roots], flags)  # C: walk, group, launch
            if r is not None:
                return batch_results(r[0], r[1], dts.pop(), lazy)
    items = [_lower_sum(e) for e in expressions]
    return run_reduce_batch(items, flags=flags, lazy=lazy)


def dot_batch(pairs, *, lazy=False) -> list:
    """[dot(x, y) for x, y in pairs] through reduce_batch (same bits).
    Pairs of plain DenseVectors of one element type and equal lengths skip
    the node objects; anything else goes through the full validation."""
    pairs = list(pairs)
    return reduce_batch([MulNode(as_node(x), as_node(y)) for x, y in pairs], lazy=lazy)


def norm2_batch(vectors, *, lazy=False) -> list:
    """[norm2(x) for x in vectors] through reduce_batch (same bits)."""
    return reduce_batch([MulNode(as_node(x), as_node(x)) for x in vectors], sqrt=True, lazy=lazy)
