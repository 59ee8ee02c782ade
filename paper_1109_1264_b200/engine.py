"""Loop engine front end: plan validation, tracing, and dispatch to the GPU.

Entry points keep the reference's signatures and validation order
(pkg/src/lanevec/engine.py:295-352):

    execute_assign(root, plan=None, *, backend=None, unroll=None,
                   packages=None, stepped=False)
    execute_reduce(...)   -> element-typed NumPy scalar
    call_trace(...)       -> [TraceEvent(kind, index, slot), ...]

`_resolve` raises every error the reference raises (LengthMismatchError,
TypeError, PlanError) before anything is launched.  After validation the
unroll plan no longer shapes the arithmetic: the tree is lowered to a postfix
signature and evaluated by ONE fused kernel (runtime.py -> libsalt.so).
Elementwise results are bit-identical to the reference for every plan (the
reference guarantees plan-invariance itself, test_acceptance.py:257-276);
reductions are compensated and deterministic, within the stated tolerance
of the reference's value for every plan.

`stepped=True` evaluates on the GPU too (the reference's stepped executor is
bit-identical to its block executor, test_engine.py:288-306); `call_trace`
returns the event sequence the reference's stepped executor records for the
same plan (engine.py:191-240) and then evaluates the tree on the GPU.
"""

from collections import namedtuple
from dataclasses import dataclass

from . import _native, runtime
from .expressions import (
    AssignNode,
    AssignReduceNode,
    FusedNode,
    Leaf,
    ScaleNode,
    SumNode,
    as_node,
    common_length,
    lower,
)
from .lanes import LaneBackend, default_backend, scalar_backend, wide_backend

__all__ = [
    "UnrollPlan",
    "PlanError",
    "select_plan",
    "masked_length",
    "execute_assign",
    "execute_reduce",
    "execute_assign_reduce",
    "execute_fused",
    "call_trace",
    "TraceEvent",
    "UNROLL_FACTORS",
    "DEFAULT_REGISTER_BUDGET",
]

UNROLL_FACTORS = (1, 2, 4, 8)
DEFAULT_REGISTER_BUDGET = 16


class PlanError(ValueError):
    """Invalid or inconsistent loop-plan configuration."""


def _pow2(n: int) -> bool:
    return n >= 1 and n & (n - 1) == 0


@dataclass(frozen=True)
class UnrollPlan:
    """Shape of one (reference) evaluation loop: unroll slots of `width`
    lanes, grouped into `packages` bursts; `masked_length` is the part the
    unrolled main loop covers (engine.py:55-95)."""

    unroll: int
    width: int
    packages: int
    masked_length: int

    def __post_init__(self):
        if self.unroll not in UNROLL_FACTORS:
            raise PlanError(f"unsupported unroll factor {self.unroll}")
        if not _pow2(self.width):
            raise PlanError(f"lane width must be a power of two, got {self.width}")
        if self.packages < 1 or self.unroll % self.packages:
            raise PlanError(f"{self.packages} packages cannot split {self.unroll} slots evenly")
        if self.masked_length < 0 or self.masked_length % self.block:
            raise PlanError(
                f"masked length {self.masked_length} is not a multiple of "
                f"{self.unroll}x{self.width}"
            )

    @property
    def block(self) -> int:
        return self.unroll * self.width

    @property
    def slots_per_package(self) -> int:
        return self.unroll // self.packages


def masked_length(length: int, unroll: int, width: int) -> int:
    """Largest multiple of unroll*width not exceeding length."""
    return length & ~(unroll * width - 1)


def select_plan(footprint: int, length: int, caps, *, unroll: int = None, packages: int = None,
                register_budget: int = None) -> UnrollPlan:
    """Largest unroll in UNROLL_FACTORS with unroll*footprint <= budget (16)
    on a packed backend, 1 on the scalar backend, unless overridden; one
    package by default (engine.py:103-145)."""
    if footprint < 1:
        raise PlanError(f"register footprint must be >= 1, got {footprint}")
    if length < 0:
        raise PlanError(f"length must be >= 0, got {length}")
    budget = DEFAULT_REGISTER_BUDGET if register_budget is None else register_budget
    if unroll is None:
        unroll = 1
        if caps.specialized:
            fitting = [u for u in UNROLL_FACTORS if u * footprint <= budget]
            unroll = max(fitting) if fitting else 1
    elif unroll not in UNROLL_FACTORS:
        raise PlanError(f"unroll override must be one of {UNROLL_FACTORS}, got {unroll}")
    packages = 1 if packages is None else packages
    return UnrollPlan(unroll, caps.width, packages, masked_length(length, unroll, caps.width))


TraceEvent = namedtuple("TraceEvent", ["kind", "index", "slot"])


def _resolve(root, plan, backend, unroll, packages):
    length = common_length(root)
    if backend is None:
        if plan is not None and plan.width == 1:
            backend = scalar_backend(root.dtype)
        elif plan is not None:
            backend = wide_backend(root.dtype, plan.width)
        else:
            backend = default_backend(root.dtype)
    elif not isinstance(backend, LaneBackend):
        raise TypeError(f"backend must be a LaneBackend, got {type(backend).__name__}")
    if backend.dtype != root.dtype:
        raise PlanError(
            f"backend element type {backend.dtype} does not match expression element type {root.dtype}"
        )
    if plan is None:
        plan = select_plan(root.register_footprint, length, backend.caps, unroll=unroll,
                           packages=packages)
    else:
        if unroll is not None or packages is not None:
            raise PlanError("pass either a prebuilt plan or overrides, not both")
        if plan.width != backend.width:
            raise PlanError(f"plan width {plan.width} does not match backend width {backend.width}")
        if plan.masked_length != masked_length(length, plan.unroll, plan.width):
            raise PlanError(
                f"plan was built for a different length (masked {plan.masked_length}, "
                f"vector length {length})"
            )
    return length, backend, plan


def _length(root, plan, backend, unroll, packages) -> int:
    """Validated length.  With no plan options the reference's default plan
    cannot fail to resolve (footprint >= 1, length >= 0, default backend of
    the tree's own dtype), so only the length check runs — the GPU never
    uses the plan."""
    if plan is None and backend is None and unroll is None and packages is None:
        return common_length(root)
    return _resolve(root, plan, backend, unroll, packages)[0]


def _trace_events(plan: UnrollPlan, length: int, reduce_root: bool) -> list:
    """The call sequence of the reference's stepped executor for `plan`:
    init, load_once per slot, per iteration and package a load burst, an op
    burst and a store burst (slot order), the scalar tail, cleanup, and the
    final reduction for reduction roots (engine.py:3-12, :191-240)."""
    ev = [TraceEvent("init", None, None)]
    ev += [TraceEvent("load_once", None, s) for s in range(plan.unroll)]
    span = plan.slots_per_package
    for i in range(0, plan.masked_length, plan.block):
        for p in range(plan.packages):
            slots = [p * span + k for k in range(span)]
            idx = [i + s * plan.width for s in slots]
            for kind in ("load", "vector_op", "store"):
                ev += [TraceEvent(kind, j, s) for j, s in zip(idx, slots)]
    ev += [TraceEvent("single_op", j, None) for j in range(plan.masked_length, length)]
    ev.append(TraceEvent("cleanup", None, None))
    if reduce_root:
        ev.append(TraceEvent("reduction", None, None))
    return ev


def _fits(lw) -> bool:
    return (len(lw.vectors) <= _native.SALT_MAX_LEAVES and len(lw.scalars) <= _native.SALT_MAX_SCALARS
            and len(lw.pscalars) <= _native.SALT_MAX_PSCALARS)


def _temporary_like(expr, length):
    """Device temporary for an intermediate of `expr`, placed like its first
    leaf (same device / same sharded partition)."""
    from .sharding import ShardedVector
    from .vectors import DenseVector

    v = next(expr.leaves()).vector
    seen = 0
    while not isinstance(v, (DenseVector, ShardedVector)) and hasattr(v, "inner") and seen < 8:
        v, seen = v.inner, seen + 1
    if isinstance(v, ShardedVector):
        return ShardedVector.zeros(length, expr.dtype, group=v.group, device=v.local.device)
    device = v.device if isinstance(v, DenseVector) else None
    return DenseVector.empty(length, expr.dtype, device=device)


def _fit(expr, length):
    """An equivalent tree that one fused kernel can take (<= SALT_MAX_LEAVES
    distinct vectors, <= SALT_MAX_SCALARS scalars, <= SALT_MAX_PSCALARS
    device scalars).  Oversized subtrees are
    evaluated on the GPU into temporaries first; every node already rounds to
    the element type, so materialising an intermediate changes no bit."""
    if _fits(lower(expr)):
        return expr
    if isinstance(expr, ScaleNode):
        child = _fit(expr.child, length)
        cand = ScaleNode(expr.alpha, child)
        return cand if _fits(lower(cand)) else ScaleNode(expr.alpha, _materialize(child, length))
    left, right = _fit(expr.left, length), _fit(expr.right, length)
    node = type(expr)
    cand = node(left, right)
    if _fits(lower(cand)):
        return cand
    # materialise the larger operand first (operand order is kept)
    if len(lower(left).tokens) >= len(lower(right).tokens):
        cand = node(_materialize(left, length), right)
    else:
        cand = node(left, _materialize(right, length))
    if _fits(lower(cand)):
        return cand
    return node(_materialize(cand.left, length), _materialize(cand.right, length))


def _materialize(expr, length):
    if isinstance(expr, Leaf):
        return expr
    tmp = _temporary_like(expr, length)
    node = Leaf(tmp)
    runtime.run_assign(lower(_fit(expr, length)), tmp, expr.dtype, length)
    return node


def _assign(root: AssignNode, length: int):
    lw = lower(root.source)
    if not _fits(lw):
        lw = lower(_fit(root.source, length))
    runtime.run_assign(lw, root.dest.vector, root.dtype, length)


def _reduce(root: SumNode, length: int, flags: int = 0, lazy: bool = False):
    lw = lower(root.child)
    if not _fits(lw):
        lw = lower(_fit(root.child, length))
    return runtime.run_reduce(lw, root.dtype, length, flags=flags, lazy=lazy)


def _check_assign_batch(statements) -> list:
    """Validate a batch of independent assignments (ops.assign_batch) as
    execute_assign would, all before anything runs; returns [(lowering,
    dest, dtype, length)].  A destination may alias its own statement's
    leaves but no other statement's operands (identity or same storage)."""
    items, dest_owner, users = [], {}, []
    for k, st in enumerate(statements):
        if not (isinstance(st, tuple) and len(st) == 2):
            raise TypeError("assign_batch takes (dest, expression) pairs")
        root = AssignNode(as_node(st[0]), as_node(st[1]))
        length = common_length(root)
        lw = lower(root.source)
        if not _fits(lw):
            lw = lower(_fit(root.source, length))
        dest = root.dest.vector
        items.append((lw, dest, root.dtype, length))
        dest_owner.setdefault(_storage_key(dest), k)
        if dest_owner[_storage_key(dest)] != k:
            raise ValueError(f"assign_batch: statements {dest_owner[_storage_key(dest)]} and {k} "
                             "write the same destination")
        users.append({_storage_key(v) for v in lw.vectors})
    for k, keys in enumerate(users):
        for key in keys:
            owner = dest_owner.get(key)
            if owner is not None and owner != k:
                raise ValueError(f"assign_batch: statement {k} reads the destination of statement {owner} "
                                 "(statements of a batch run concurrently)")
    return items


def _lower_sum(expression):
    """(lowering, dtype, length) of sum(expression), validated as
    execute_reduce validates it (reduce_batch)."""
    root = SumNode(as_node(expression))
    length = common_length(root)
    lw = lower(root.child)
    if not _fits(lw):
        lw = lower(_fit(root.child, length))
    return lw, root.dtype, length


def _storage_key(v):
    t = getattr(v, "_data", None)
    return ("ptr", t.get_device(), t.data_ptr()) if t is not None and t.numel() else ("id", id(v))


def execute_assign(root, plan: UnrollPlan = None, *, backend: LaneBackend = None,
                   unroll: int = None, packages: int = None, stepped: bool = False) -> None:
    """Evaluate an assignment tree, writing every destination element once."""
    if not isinstance(root, AssignNode):
        raise TypeError("execute_assign requires an assignment root")
    if plan is None and backend is None and unroll is None and packages is None:
        fast = _native.fastpath()
        if fast is not None and fast.assign(root.dest.vector, root.source):
            return
    _assign(root, _length(root, plan, backend, unroll, packages))


def execute_reduce(root, plan: UnrollPlan = None, *, backend: LaneBackend = None,
                   unroll: int = None, packages: int = None, stepped: bool = False,
                   lazy: bool = False, _flags: int = 0):
    """Evaluate a reduction tree; returns an element-typed NumPy scalar
    (or a DeviceScalar without host synchronisation when lazy=True)."""
    if not isinstance(root, SumNode):
        raise TypeError("execute_reduce requires a reduction root")
    if plan is None and backend is None and unroll is None and packages is None:
        fast = _native.fastpath()
        if fast is not None:
            r = fast.reduce(root.child, _flags, lazy)
            if r is not None:
                return r
    return _reduce(root, _length(root, plan, backend, unroll, packages), flags=_flags, lazy=lazy)


def execute_assign_reduce(root, plan: UnrollPlan = None, *, backend: LaneBackend = None,
                          unroll: int = None, packages: int = None, stepped: bool = False,
                          lazy: bool = False, _flags: int = 0):
    """Evaluate an AssignReduceNode in one pass: assign, then return the sum
    over the freshly assigned values (e.g. axpy then dot, BASELINE config 5)."""
    if not isinstance(root, AssignReduceNode):
        raise TypeError("execute_assign_reduce requires an AssignReduceNode root")
    if plan is None and backend is None and unroll is None and packages is None:
        fast = _native.fastpath()
        if fast is not None:
            r = fast.assign_reduce(root.assign.dest.vector, root.assign.source, root.total.child,
                                   _flags, lazy)
            if r is not None:
                return r
    length = _length(root, plan, backend, unroll, packages)
    lwa = lower(root.assign.source)
    lwr = lower(root.total.child, parent=lwa, dest=root.assign.dest.vector)
    if not _fits(lwa):
        # too large for one fused kernel: assign, then reduce over the new values
        _assign(root.assign, length)
        return _reduce(root.total, length, flags=_flags, lazy=lazy)
    return runtime.run_assign_reduce(lwa, lwr, root.assign.dest.vector, root.dtype, length,
                                     flags=_flags, lazy=lazy)


def execute_fused(root, *, lazy: bool = False, _flags: int = 0):
    """Evaluate a FusedNode: all its assignments (and its final reduction,
    whose value is returned) in ONE pass when every vector is a plain device
    DenseVector and the statements fit one kernel; otherwise statement by
    statement — the same results either way."""
    if not isinstance(root, FusedNode):
        raise TypeError("execute_fused requires a FusedNode root")
    if root.assigns and len(root.assigns) <= _native.SALT_MAX_ROOTS:
        fast = _native.fastpath()
        if fast is not None:
            r = fast.fused(tuple((s.dest.vector, s.source) for s in root.assigns),
                           None if root.total is None else root.total.child, _flags, lazy)
            if r is not None:
                return r[0]
    length = common_length(root)
    if len(root.assigns) <= _native.SALT_MAX_ROOTS:
        asig, rsig, lw, dests = root.lower()
        if _fits(lw):
            handled, result = runtime.run_fused(asig, rsig, lw, dests, root.dtype, length,
                                                flags=_flags, lazy=lazy)
            if handled:
                return result
    for s in root.assigns:
        _assign(s, length)
    if root.total is not None:
        return _reduce(root.total, length, flags=_flags, lazy=lazy)
    return None


def call_trace(root, plan: UnrollPlan = None, *, backend: LaneBackend = None,
               unroll: int = None, packages: int = None) -> list:
    """Evaluate `root` and return the reference stepped executor's event
    sequence for the resolved plan."""
    length, _, plan = _resolve(root, plan, backend, unroll, packages)
    is_reduce = isinstance(root, SumNode)
    if is_reduce:
        _reduce(root, length)
    elif isinstance(root, AssignNode):
        _assign(root, length)
    else:
        raise TypeError("call_trace requires an assignment or reduction root")
    return _trace_events(plan, length, is_reduce)
