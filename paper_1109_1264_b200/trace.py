"""Device-observed evaluation traces.

The reference's stepped executor records its contract calls in order
(call_trace, /root/reference/pkg/src/lanevec/engine.py:191-240, :332-352):
per package of unroll slots a load burst, an op burst and a store burst,
then the scalar tail.  `call_trace` here returns that event list for the
resolved plan (engine._trace_events).  `device_trace` instead OBSERVES the
GPU: it evaluates the tree once with the NVRTC build of its kernel compiled
with -DSALT_TRACE (salt_set_trace, include/salt.h), in which thread 0 of the
first streaming CTA appends every event it executes to a device buffer —
its load burst per tile (all UNR slots' vectors issued before any
arithmetic), the evaluation and store of each slot, its scalar head/tail
elements and, for reductions, the point where its partial joins the CTA's.
The element indices are real: thread 0's slot u of tile t covers the V
elements starting at head + (t*BLOCK*UNR + u*BLOCK)*V.  The results of the
traced evaluation are the same bits as the untraced one.
"""

from collections import namedtuple

import torch

from . import _native
from .engine import TraceEvent, _assign, _reduce
from .expressions import AssignNode, SumNode, common_length

__all__ = ["device_trace", "DeviceTrace"]

KINDS = {0: "load", 1: "vector_op", 2: "store", 3: "single_op", 4: "reduction"}

DeviceTrace = namedtuple("DeviceTrace", ["events", "truncated", "result"])


def device_trace(root, capacity: int = 1 << 16) -> DeviceTrace:
    """Evaluate `root` (an AssignNode or SumNode over device vectors) once
    and return the events one GPU thread executed, as TraceEvent(kind,
    element index, slot) tuples (index / slot None where they do not apply),
    whether the buffer overflowed, and the reduction's value (None for an
    assignment)."""
    if not isinstance(root, (AssignNode, SumNode)):
        raise TypeError("device_trace requires an assignment or reduction root")
    length = common_length(root)
    dev = None
    for leaf in root.leaves():
        t = getattr(leaf.vector, "tensor", None)
        if t is not None and t.device.type == "cuda":
            dev = t.device
            break
    if dev is None:
        raise TypeError("device_trace needs device-resident DenseVector operands")
    buf = torch.zeros(1 + 3 * capacity, dtype=torch.int64, device=dev)
    lib = _native.lib()
    _native.check(lib.salt_set_trace(buf.data_ptr(), buf.numel()))
    result = None
    try:
        if isinstance(root, SumNode):
            result = _reduce(root, length)
        else:
            _assign(root, length)
        torch.cuda.synchronize(dev)
    finally:
        lib.salt_set_trace(None, 0)
    host = buf.cpu()
    count = int(host[0])
    rows = host[1:1 + 3 * min(count, capacity)].view(-1, 3).tolist()
    events = [TraceEvent(KINDS[k], None if i < 0 else int(i), None if s < 0 else int(s)) for k, i, s in rows]
    return DeviceTrace(events, count >= capacity, result)
