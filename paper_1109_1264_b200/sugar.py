"""Operator sugar shared by the vector types (DenseVector, CountingVector,
ShardedVector).

Arithmetic on vectors only builds lazy expression nodes — nothing is read
until an assignment or a sum runs the fused kernel (reference
vectors.py:109-138, criterion 5).  `vector * number` and `number * vector`
scale; `-vector` scales by -1.  There is deliberately no reflected + / -:
`number + vector` stays a TypeError, as in the reference
(test_expressions.py:51-56).
"""

__all__ = ["VectorOps"]


def _nodes():
    from . import expressions  # late: expressions imports the vector types

    return expressions


class VectorOps:
    __slots__ = ()

    def __add__(self, other):
        return _nodes().add_nodes(self, other)

    def __sub__(self, other):
        return _nodes().sub_nodes(self, other)

    def __mul__(self, other):
        return _nodes().mul_nodes(self, other)

    def __rmul__(self, other):
        return _nodes().scale_node(other, self)

    def __neg__(self):
        return _nodes().negate_node(self)
