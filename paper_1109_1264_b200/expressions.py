"""Lazy expression nodes built by operator overloading.

Same classes, constructors, checks and operator sugar as the reference
(pkg/src/lanevec/expressions.py): building a tree touches no element
(test_acceptance.py:246-254); dtype mismatches are TypeErrors
at construction (:196-203, :340-343); ScaleNode coerces alpha to the element
type (:282); AssignNode's destination must be a Leaf (:338-339); lengths are
checked before any access (`common_length`, :483-497).

What differs is evaluation.  The reference nodes implement a per-block CPU
contract (init / load / vector_op / store / single_op ..., :3-15) that its
Python loop engine drives.  Here every node instead knows how to emit itself
in postfix (`_postfix`), so the engine can lower the whole tree to one
signature string — e.g. `S0 L0 * S1 L1 L2 - * +` for alpha*a + beta*(b - c)
— and hand it to libsalt.so, which runs the tree as ONE fused sm_100a kernel.
"""

import numbers

import numpy as np

from .lanes import LaneVector, horizontal_sum
from .vectors import DenseVector, DeviceScalar

__all__ = [
    "Expression",
    "Leaf",
    "AddNode",
    "SubNode",
    "MulNode",
    "ScaleNode",
    "AssignNode",
    "SumNode",
    "AssignReduceNode",
    "FusedNode",
    "LengthMismatchError",
    "Cell",
    "SlotCell",
    "as_node",
    "common_length",
    "combine_partials",
    "traffic",
]


class LengthMismatchError(ValueError):
    """Leaves of one expression tree disagree on length."""


def _is_vector(obj) -> bool:
    # The reference's duck-typed vector test (expressions.py:68-69).
    return hasattr(obj, "read_block") and hasattr(obj, "dtype")


def as_node(obj) -> "Expression":
    """Wrap a vector in a Leaf; pass expressions through."""
    if type(obj) is DenseVector:
        return Leaf(obj)
    if isinstance(obj, Expression):
        return obj
    if _is_vector(obj):
        return Leaf(obj)
    raise TypeError(f"cannot use {type(obj).__name__} in a vector expression")


def add_nodes(a, b):
    return AddNode(as_node(a), as_node(b))


def sub_nodes(a, b):
    return SubNode(as_node(a), as_node(b))


def mul_nodes(a, b):
    if isinstance(b, (numbers.Real, DeviceScalar)):
        return ScaleNode(b, as_node(a))
    return MulNode(as_node(a), as_node(b))


def scale_node(alpha, x):
    return ScaleNode(alpha, as_node(x))


def negate_node(x):
    return ScaleNode(-1, as_node(x))


class _Lowering:
    """Collects leaves (deduplicated by vector identity, numbered by first
    appearance in postfix order) and scalars (numbered by appearance)."""

    __slots__ = ("tokens", "vectors", "_ids", "scalars", "occurrences", "dests", "pscalars")

    def __init__(self, parent: "_Lowering" = None, dest=None, dests=None):
        # A child lowering (a later tree of the same fused kernel) shares the
        # parent's leaf table and scalar list; its references to a vector
        # assigned earlier in the kernel become `D<k>`, the value root k has
        # just computed (`dest` alone is root 0).
        self.tokens = []
        self.vectors = parent.vectors if parent else []
        self._ids = parent._ids if parent else {}
        self.scalars = parent.scalars if parent else []
        self.occurrences = parent.occurrences if parent else []
        self.pscalars = parent.pscalars if parent else []  # DeviceScalar operands
        self.dests = dict(dests or {})
        if dest is not None:
            self.dests[id(dest)] = 0

    def leaf(self, vector):
        k = self.dests.get(id(vector))
        if k is not None:
            self.tokens.append(f"D{k}")
            return
        k = self._ids.get(id(vector))
        if k is None:
            k = len(self.vectors)
            self._ids[id(vector)] = k
            self.vectors.append(vector)
            self.occurrences.append(0)
        self.occurrences[k] += 1
        self.tokens.append(f"L{k}")

    def scalar(self, value):
        if isinstance(value, DeviceScalar):
            # read by the kernel from device memory: no host round trip
            self.tokens.append(f"P{len(self.pscalars)}")
            self.pscalars.append(value)
            return
        self.tokens.append(f"S{len(self.scalars)}")
        self.scalars.append(float(value))


class SlotCell:
    """One lane register of a node (reference expressions.py:49-57): in the
    fused kernel, the V-lane register a leaf is loaded into, the broadcast
    scalar of a ScaleNode, an assigned value or a reduction accumulator."""

    __slots__ = ("backend", "value")

    def __init__(self, backend):
        self.backend, self.value = backend, None


class Cell:
    """One loop-wide scalar (reference expressions.py:59-66): the remainder
    accumulator of a SumNode (the kernel's scalar head/tail sum)."""

    __slots__ = ("value",)

    def __init__(self):
        self.value = None


def _storage(node, backend):
    """Per-slot register layout of `node`, mirroring the tree: a SlotCell
    per register, a pair for a binary node, (own register, child layout)
    for Scale / Assign / Sum (reference contract: expressions.py:166-167,
    213-214, 291-292, 360-361, 425-426)."""
    if isinstance(node, Leaf):
        return SlotCell(backend)
    if isinstance(node, _BinaryNode):
        return (_storage(node.left, backend), _storage(node.right, backend))
    inner = {ScaleNode: "child", SumNode: "child", AssignNode: "source"}.get(type(node))
    if inner is None:
        raise TypeError(f"{type(node).__name__} has no per-slot storage")
    return (SlotCell(backend), _storage(getattr(node, inner), backend))


def _temporary(node, backend):
    """Loop-wide scalars of `node`: only a SumNode owns one (its remainder
    Cell); other nodes pass their children's through (reference
    expressions.py:169-170, 216-217, 294-295, 363-364, 428-429)."""
    if isinstance(node, Leaf):
        return None
    if isinstance(node, _BinaryNode):
        return (_temporary(node.left, backend), _temporary(node.right, backend))
    if isinstance(node, SumNode):
        return (Cell(), _temporary(node.child, backend))
    if isinstance(node, ScaleNode):
        return _temporary(node.child, backend)
    if isinstance(node, AssignNode):
        return _temporary(node.source, backend)
    raise TypeError(f"{type(node).__name__} has no temporary storage")


class Expression:
    """Base class: operator sugar (reference expressions.py:103-132)."""

    __slots__ = ()

    __array_ufunc__ = None

    def make_storage(self, backend):
        return _storage(self, backend)

    def make_temporary(self, backend):
        return _temporary(self, backend)

    def __add__(self, other):
        return add_nodes(self, other)

    def __radd__(self, other):
        return add_nodes(other, self)

    def __sub__(self, other):
        return sub_nodes(self, other)

    def __rsub__(self, other):
        return sub_nodes(other, self)

    def __mul__(self, other):
        return mul_nodes(self, other)

    def __rmul__(self, other):
        if isinstance(other, (numbers.Real, DeviceScalar)):
            return ScaleNode(other, self)
        return mul_nodes(other, self)

    def __neg__(self):
        return negate_node(self)


class Leaf(Expression):
    """Direct view of a vector."""

    __slots__ = ("vector", "dtype")

    def __init__(self, vector):
        self.vector = vector
        self.dtype = vector.dtype

    @property
    def register_footprint(self) -> int:
        return 1

    def leaves(self):
        yield self

    def _postfix(self, lw: _Lowering):
        lw.leaf(self.vector)

    def __repr__(self):
        return f"Leaf({self.vector!r})"


class _BinaryNode(Expression):
    """left (op) right, one IEEE op in the element type, left operand first."""

    __slots__ = ("left", "right", "dtype")

    _symbol = "?"

    def __init__(self, left: Expression, right: Expression):
        if left.dtype != right.dtype:
            raise TypeError(f"mixed element types in expression: {left.dtype} vs {right.dtype}")
        self.left = left
        self.right = right
        self.dtype = left.dtype

    @property
    def register_footprint(self) -> int:
        return self.left.register_footprint + self.right.register_footprint

    def leaves(self):
        yield from self.left.leaves()
        yield from self.right.leaves()

    def _postfix(self, lw: _Lowering):
        self.left._postfix(lw)
        self.right._postfix(lw)
        lw.tokens.append(self._symbol)

    def __repr__(self):
        return f"({self.left!r} {self._symbol} {self.right!r})"


class AddNode(_BinaryNode):
    __slots__ = ()
    _symbol = "+"


class SubNode(_BinaryNode):
    __slots__ = ()
    _symbol = "-"


class MulNode(_BinaryNode):
    __slots__ = ()
    _symbol = "*"


class ScaleNode(Expression):
    """alpha * child; alpha coerced to the element type at construction."""

    __slots__ = ("alpha", "child", "dtype")

    def __init__(self, alpha, child: Expression):
        self.child = child
        self.dtype = child.dtype
        if isinstance(alpha, DeviceScalar):
            # a device-resident alpha is already element-typed; keep it there
            if alpha.dtype != self.dtype:
                raise TypeError(f"mixed element types: scalar {alpha.dtype} vs {self.dtype}")
            self.alpha = alpha
        else:
            self.alpha = self.dtype.type(alpha)

    @property
    def register_footprint(self) -> int:
        return 1 + self.child.register_footprint

    def leaves(self):
        yield from self.child.leaves()

    def _postfix(self, lw: _Lowering):
        # alpha is the LEFT operand, as in the reference (expressions.py:320)
        lw.scalar(self.alpha)
        self.child._postfix(lw)
        lw.tokens.append("*")

    def __repr__(self):
        a = "device" if isinstance(self.alpha, DeviceScalar) else repr(float(self.alpha))
        return f"({a} * {self.child!r})"


class AssignNode(Expression):
    """Evaluation root writing an elementwise expression into `dest`.

    The destination is written once per element and never read unless it
    is also a source leaf; exact aliasing (dest is a source leaf, e.g. scal
    and axpy) is safe because each thread computes its whole vector of
    results before storing it.  Overlap at a shifted offset is unsupported
    and unchecked, as in the reference (expressions.py:326-333).
    """

    __slots__ = ("dest", "source", "dtype")

    def __init__(self, dest: Leaf, source: Expression):
        if not isinstance(dest, Leaf):
            raise TypeError("assignment destination must be a vector leaf")
        if dest.dtype != source.dtype:
            raise TypeError(f"mixed element types in assignment: {dest.dtype} vs {source.dtype}")
        self.dest = dest
        self.source = source
        self.dtype = dest.dtype

    @property
    def register_footprint(self) -> int:
        # +1 lane for the result held between op burst and store burst
        # (reference expressions.py:350-354; only plan selection uses it).
        return 1 + self.source.register_footprint

    def leaves(self):
        yield self.dest
        yield from self.source.leaves()

    def __repr__(self):
        return f"Assign({self.dest!r} <- {self.source!r})"


class SumNode(Expression):
    """Reduction root: sum of the child over all indices."""

    __slots__ = ("child", "dtype")

    def __init__(self, child: Expression):
        self.child = child
        self.dtype = child.dtype

    @property
    def register_footprint(self) -> int:
        return 1 + self.child.register_footprint

    def leaves(self):
        yield from self.child.leaves()

    def __repr__(self):
        return f"Sum({self.child!r})"


def combine_partials(rows, remainder):
    """The reference's fixed fold of lane accumulators (expressions.py:470-480):
    rows in order, each folded left to right, remainder last.  Kept for API
    parity; GPU reductions combine double-double partials instead."""
    total = None
    for row in rows:
        h = horizontal_sum(LaneVector(np.asarray(row)))
        total = h if total is None else total + h
    return remainder if total is None else total + remainder


def common_length(root: Expression) -> int:
    """Length shared by every leaf (the destination included); checked before
    any element is touched.  Leaves are visited in the reference's order
    (destination first, then left to right), so the first mismatch reported
    is the same one the reference reports."""
    length = None
    stack = [root]
    while stack:
        node = stack.pop()
        if isinstance(node, Leaf):
            n = len(node.vector)
            if length is None:
                length = n
            elif n != length:
                raise LengthMismatchError(f"expression mixes vectors of length {length} and {n}")
            continue
        if isinstance(node, _BinaryNode):
            stack.append(node.right)
            stack.append(node.left)
        elif isinstance(node, (ScaleNode, SumNode)):
            stack.append(node.child)
        elif isinstance(node, AssignNode):
            stack.append(node.source)
            stack.append(node.dest)
        else:  # AssignReduceNode and any other composite root
            stack.extend(reversed(list(node.leaves())))
    if length is None:
        raise TypeError("expression has no vector leaves")
    return length


class AssignReduceNode(Expression):
    """Fused root: run `assign`, then reduce `total` over the NEW values of
    the destination, in one pass over memory (no reference counterpart: the
    reference needs two traversals, ops.axpy then ops.dot, ops.py:18-36).

    Inside `total`, leaves that are the destination vector read the value
    just assigned; every other leaf reads its (unchanged) input.
    """

    __slots__ = ("assign", "total", "dtype")

    def __init__(self, assign: AssignNode, total: SumNode):
        if not isinstance(assign, AssignNode):
            raise TypeError("AssignReduceNode needs an AssignNode")
        if not isinstance(total, SumNode):
            raise TypeError("AssignReduceNode needs a SumNode")
        if assign.dtype != total.dtype:
            raise TypeError(f"mixed element types: {assign.dtype} vs {total.dtype}")
        self.assign = assign
        self.total = total
        self.dtype = assign.dtype

    @property
    def register_footprint(self) -> int:
        return self.assign.register_footprint + self.total.register_footprint

    def leaves(self):
        yield from self.assign.leaves()
        yield from self.total.leaves()

    def __repr__(self):
        return f"AssignReduce({self.assign!r}; {self.total!r})"


def lower(expr: Expression, parent: _Lowering = None, dest=None, dests=None) -> _Lowering:
    """Postfix signature of an elementwise tree (leaves + scalars collected)."""
    lw = _Lowering(parent, dest, dests)
    expr._postfix(lw)
    return lw


class FusedNode(Expression):
    """Several statements evaluated in ONE pass over memory: up to four
    assignments and optionally one final reduction (no reference
    counterpart — the reference runs one traversal per statement).

    Per element the statements run in order, so the results are exactly
    those of running them one after another: a statement that reads a
    vector assigned by an earlier statement sees the new value (the kernel
    reads it from registers, not memory).  Example, one conjugate-gradient
    update:

        FusedNode([AssignNode(x, x + a*p), AssignNode(r, r - a*q)], SumNode(r*r))
    """

    __slots__ = ("assigns", "total", "dtype")

    def __init__(self, assigns, total=None):
        assigns = list(assigns)
        if not assigns or not all(isinstance(s, AssignNode) for s in assigns):
            raise TypeError("FusedNode needs one or more AssignNode statements")
        if total is not None and not isinstance(total, SumNode):
            raise TypeError("the final statement of a FusedNode must be a SumNode")
        dts = {s.dtype for s in assigns} | ({total.dtype} if total is not None else set())
        if len(dts) != 1:
            raise TypeError(f"mixed element types in fused statements: {sorted(map(str, dts))}")
        self.assigns = assigns
        self.total = total
        self.dtype = assigns[0].dtype

    @property
    def register_footprint(self) -> int:
        fp = sum(s.register_footprint for s in self.assigns)
        return fp + (self.total.register_footprint if self.total is not None else 0)

    def leaves(self):
        for s in self.assigns:
            yield from s.leaves()
        if self.total is not None:
            yield from self.total.leaves()

    def lower(self):
        """(assign signature with roots joined by ' ; ', reduce signature or
        None, shared _Lowering, destination vectors)."""
        lw = _Lowering()
        parts, dests, written = [], [], {}
        for k, s in enumerate(self.assigns):
            sub = lower(s.source, parent=lw, dests=written)
            parts.append(" ".join(sub.tokens))
            dests.append(s.dest.vector)
            written[id(s.dest.vector)] = k
        rsig = None
        if self.total is not None:
            rsig = " ".join(lower(self.total.child, parent=lw, dests=written).tokens)
        return " ; ".join(parts), rsig, lw, dests

    def __repr__(self):
        body = "; ".join(repr(s) for s in self.assigns)
        return f"Fused({body}" + (f"; {self.total!r})" if self.total is not None else ")")


def traffic(root: Expression) -> dict:
    """Static traffic of one fused evaluation of `root` — the GPU analogue of
    the reference's CountingVector fusion checks (test_acceptance.py:222-243):
    every DISTINCT vector read is loaded once (a destination that is also a
    source leaf counts as a read), the destination is stored once.  These are
    the algorithmic bytes the roofline numbers are computed from."""
    n = common_length(root)
    if isinstance(root, AssignNode):
        lw, dest = lower(root.source), root.dest.vector
    elif isinstance(root, SumNode):
        lw, dest = lower(root.child), None
    elif isinstance(root, AssignReduceNode):
        lw, dest = lower(root.assign.source), root.assign.dest.vector
        lower(root.total.child, parent=lw, dest=dest)
    else:
        raise TypeError("traffic() needs an AssignNode, SumNode or AssignReduceNode root")
    reads = len(lw.vectors)
    writes = 1 if dest is not None else 0
    size = root.dtype.itemsize
    return {
        "vectors_read": reads,
        "vectors_written": writes,
        "elements": n,
        "bytes": size * n * (reads + writes),
    }
