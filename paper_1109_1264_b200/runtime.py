"""Execution of lowered trees through libsalt.so.

The reference's hot loops (engine.py:243-292) become one C-ABI call each:

  device operands  -> salt_assign / salt_reduce / salt_assign_reduce on the
                      caller's current CUDA stream (asynchronous for assign;
                      reductions synchronise only to return the host scalar,
                      or not at all with lazy=True)
  host operands    -> salt_assign_host / salt_reduce_host (pinned host memory
                      streamed through the GPU, blocking)
  sharded operands -> each rank evaluates its own block; reductions
                      all-gather the per-rank double-double partials and
                      combine them in rank order (sharding.py)

The common case — plain device DenseVectors — takes a fast path (no
placement object, raw stream handle, array.array argument buffers): the
Python cost of one call is about 10 us on top of the ~3 us kernel launch.
Anything else goes through `Placement`, which resolves each operand to its
storage: a DenseVector itself, the inner vector of a CountingVector, the
local block of a ShardedVector, or — for any other duck-typed vector
(expressions.py:68-69) — a temporary device copy made through its
read_block/write_block protocol.
"""

import array
import ctypes
import threading

import numpy as np
import torch

from . import _native
from .lanes import as_dtype
from .vectors import DenseVector, DeviceScalar

__all__ = ["run_assign", "run_reduce", "run_assign_reduce", "run_fused", "run_assign_batch", "run_reduce_batch",
           "Placement"]

_ws_lock = threading.Lock()
_workspaces = {}
_capture_workspaces = {}
try:
    _is_capturing = torch._C._cuda_isCurrentStreamCapturing
except AttributeError:  # pragma: no cover
    _is_capturing = torch.cuda.is_current_stream_capturing
_host_state = {}
_HOST_STAGING_BYTES = 768 << 20

try:  # raw cudaStream_t of the current stream, ~10x cheaper than the public API
    _raw_stream = torch._C._cuda_getCurrentRawStream
except AttributeError:  # pragma: no cover
    def _raw_stream(index):
        return torch.cuda.current_stream(index).cuda_stream


def _dtype_code(dt) -> int:
    return _native.SALT_F32 if dt.itemsize == 4 else _native.SALT_F64


class _OnDevice:
    """Make `index` the current CUDA device for the call (no-op if it is)."""

    __slots__ = ("index", "prev")

    def __init__(self, index):
        self.index = index
        self.prev = None

    def __enter__(self):
        cur = torch.cuda.current_device()
        if cur != self.index:
            self.prev = cur
            torch.cuda.set_device(self.index)
        return self

    def __exit__(self, *exc):
        if self.prev is not None:
            torch.cuda.set_device(self.prev)


def _fast(vectors, dest):
    """(device index, leaf pointers, dest pointer) when every operand is a
    plain device DenseVector on one device; None otherwise."""
    dev = None
    ptrs = []
    for v in vectors:
        if type(v) is not DenseVector:
            return None
        t = v._data
        d = t.get_device()
        if d < 0 or (dev is not None and d != dev):
            return None
        dev = d
        ptrs.append(t.data_ptr())
    dptr = 0
    if dest is not None:
        if type(dest) is not DenseVector:
            return None
        t = dest._data
        d = t.get_device()
        if d < 0 or (dev is not None and d != dev):
            return None
        dev = d
        dptr = t.data_ptr()
    if dev is None:
        return None
    return dev, ptrs, dptr


def _unwrap(vec):
    """Storage DenseVector behind `vec` (or None for a foreign duck vector)."""
    seen = 0
    while not isinstance(vec, DenseVector):
        inner = getattr(vec, "inner", None)
        if inner is None or seen > 8:
            return None
        vec, seen = inner, seen + 1
    return vec


def _shard_of(v):
    from .sharding import ShardedVector

    seen = 0
    while not isinstance(v, ShardedVector) and seen < 8:
        inner = getattr(v, "inner", None)
        if inner is None:
            return v
        v, seen = inner, seen + 1
    return v


class Placement:
    """Where a lowered tree runs, and the storage of each operand."""

    __slots__ = ("kind", "device", "leaves", "dest", "sharded", "staged_dest", "n")

    def __init__(self, vectors, dest, n):
        from .sharding import ShardedVector

        self.sharded = None
        self.staged_dest = None
        self.n = n
        everything = list(vectors) + ([dest] if dest is not None else [])
        shard_flags = [isinstance(_shard_of(v), ShardedVector) for v in everything]
        if any(shard_flags):
            if not all(shard_flags):
                raise TypeError("cannot mix sharded and unsharded vectors in one expression")
            shards = [_shard_of(v) for v in everything]
            first = shards[0]
            for s in shards[1:]:
                if not first.same_partition(s):
                    raise ValueError("sharded vectors in one expression must share a partition")
            self.sharded = first
            self.n = len(first.local)
            storage = [s.local for s in shards]
        else:
            storage = [_unwrap(v) for v in everything]
        # Foreign duck vectors: stage through a device copy.
        dev = next((s.device for s in storage if s is not None and s.device.type == "cuda"), None)
        if dev is None and any(s is None for s in storage):
            dev = _require_cuda()
        for i, s in enumerate(storage):
            if s is None:
                v = everything[i]
                staged = DenseVector.from_values(v.read_block(0, len(v)), v.dtype, device=dev)
                storage[i] = staged
                if dest is not None and i == len(everything) - 1:
                    self.staged_dest = (v, staged)
        devices = {s.device for s in storage}
        if len(devices) != 1:
            raise ValueError(
                "all vectors of one expression must live on the same device, got "
                + ", ".join(sorted(str(d) for d in devices))
            )
        self.device = devices.pop()
        self.kind = "host" if self.device.type == "cpu" else "device"
        if dest is not None:
            self.dest = storage[-1]
            self.leaves = storage[:-1]
        else:
            self.dest = None
            self.leaves = storage

    @property
    def pointers(self):
        return [s.tensor.data_ptr() for s in self.leaves]

    @property
    def dest_pointer(self):
        return self.dest.tensor.data_ptr() if self.dest is not None else 0

    def finish(self):
        if self.staged_dest is not None:
            v, staged = self.staged_dest
            v.write_block(0, len(v), staged.to_array())


def _require_cuda() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError(
            "no CUDA device: paper_1109_1264_b200 evaluates expressions on the GPU only "
            "(there is no CPU evaluation path)"
        )
    return torch.device("cuda", torch.cuda.current_device())


_MAX_CACHED_WORKSPACES = 64


def _capture_workspace(index: int, stream_ptr: int) -> torch.Tensor:
    """Private scratch of the CUDA graph being captured on `stream_ptr`: the
    graph bakes the workspace address in, so two graphs replayed at once on
    different streams — or a graph replayed while eager reductions run on
    its capture stream — must not share tickets.  One workspace per capture
    (all reductions of one captured stream run in order), allocated in the
    graph's memory pool and kept for the life of the process; its ticket
    words are zeroed by a captured memset, i.e. at the start of every
    replay."""
    cid = _native.lib().salt_capture_id(stream_ptr)
    key = (index, stream_ptr, cid)
    ws = _capture_workspaces.get(key)
    if ws is None:
        nbytes = _native.lib().salt_reduce_workspace_bytes() + 256
        ws = torch.empty(nbytes, dtype=torch.uint8, device=torch.device("cuda", index))
        ws[: _native.SALT_WORKSPACE_TICKET_BYTES].zero_()
        _capture_workspaces[key] = ws
    return ws


def _workspace(index: int, stream_ptr: int) -> torch.Tensor:
    """Reduction scratch of (device, stream): zeroed once, then kept — the
    kernels reset their tickets themselves, so consecutive reductions on one
    stream share it safely.  Beyond _MAX_CACHED_WORKSPACES streams a fresh
    scratch is made per call (tickets zeroed, tied to the stream).  While
    the stream is being captured into a CUDA graph: the capture's own
    scratch (_capture_workspace)."""
    if _is_capturing():
        return _capture_workspace(index, stream_ptr)
    key = (index, stream_ptr)
    ws = _workspaces.get(key)
    if ws is None:
        with _ws_lock:
            ws = _workspaces.get(key)
            if ws is None:
                # + 256 bytes: the C fast path's result slot (csrc/fastpath.c)
                nbytes = _native.lib().salt_reduce_workspace_bytes() + 256
                device = torch.device("cuda", index)
                if len(_workspaces) < _MAX_CACHED_WORKSPACES:
                    ws = torch.zeros(nbytes, dtype=torch.uint8, device=device)
                    _workspaces[key] = ws
                else:
                    ws = torch.empty(nbytes, dtype=torch.uint8, device=device)
                    ws[: _native.SALT_WORKSPACE_TICKET_BYTES].zero_()
                    ws.record_stream(torch.cuda.current_stream(device))
    return ws


def _lazy_out(index: int, code: int):
    """(DeviceScalar, device pointer) for a lazy reduction result (C fast path)."""
    out = torch.empty(1, dtype=torch.float64, device=torch.device("cuda", index))
    dt = np.dtype(np.float32 if code == _native.SALT_F32 else np.float64)
    return _result(dt, out, None, True), out.data_ptr()


def _host_resources(device: torch.device):
    st = _host_state.get(device.index)
    if st is None:
        with _ws_lock:
            st = _host_state.get(device.index)
            if st is None:
                staging = torch.empty(_HOST_STAGING_BYTES, dtype=torch.uint8, device=device)
                streams = [torch.cuda.Stream(device=device) for _ in range(3)]
                st = (threading.Lock(), staging, streams)
                _host_state[device.index] = st
    return st


def _record_counts(lw, dest, n):
    """CountingVector bookkeeping: each leaf OCCURRENCE reads n elements and
    the destination is written n times (reference semantics, test_engine.py
    :468-485), even though the fused kernel loads a repeated leaf once."""
    for vec, occ in zip(lw.vectors, lw.occurrences):
        if hasattr(vec, "read_count"):
            vec.read_count += occ * n
    if dest is not None and hasattr(dest, "write_count"):
        dest.write_count += n


def _host_call(fn):
    """Run a blocking host-streaming call with the device's staging area and
    three streams (serialised per device)."""
    dev = _require_cuda()
    lock, staging, streams = _host_resources(dev)
    with lock, _OnDevice(dev.index):
        sptrs, keep = _native.ptr_array([s.cuda_stream for s in streams])
        torch.cuda.current_stream(dev).synchronize()
        _native.check(fn(staging.data_ptr(), staging.numel(), sptrs))
        del keep


# ---------------------------------------------------------------- assign
def run_assign(lw, dest, dtype, n):
    if lw.pscalars:
        handled, _ = run_fused(" ".join(lw.tokens), None, lw, [dest], dtype, n)
        return _device_scalars_only(handled)
    lib = _native.lib()
    code = _dtype_code(dtype)
    sig = " ".join(lw.tokens).encode()
    scal, keep_s = _native.double_array(lw.scalars)
    nl, ns = len(lw.vectors), len(lw.scalars)
    fast = _fast(lw.vectors, dest)
    if fast is not None:
        dev, ptrs, dptr = fast
        leaves, keep_l = _native.ptr_array(ptrs)
        if torch.cuda.current_device() == dev:
            _native.check(lib.salt_assign(code, sig, dptr, leaves, nl, scal, ns, n, _raw_stream(dev)))
        else:
            with _OnDevice(dev):
                _native.check(lib.salt_assign(code, sig, dptr, leaves, nl, scal, ns, n, _raw_stream(dev)))
        return
    pl = Placement(lw.vectors, dest, n)
    leaves, keep_l = _native.ptr_array(pl.pointers)
    if pl.kind == "host":
        if pl.n:
            _host_call(lambda st, sb, sp: lib.salt_assign_host(
                code, sig, pl.dest_pointer, leaves, nl, scal, ns, pl.n, st, sb, sp))
    else:
        with _OnDevice(pl.device.index):
            _native.check(lib.salt_assign(code, sig, pl.dest_pointer, leaves, nl, scal, ns, pl.n,
                                          _raw_stream(pl.device.index)))
    pl.finish()
    _record_counts(lw, dest, n)


def run_assign_batch(items):
    """items: [(lowering, dest, dtype, n)] of validated assignments.  Those
    whose operands are plain device DenseVectors are grouped by (device,
    element type, signature) and each group goes to salt_assign_batch (one
    launch per up to 96 problems); the rest run one by one.  Returns the
    number of statements that went through a batch."""
    groups, rest = {}, []
    for lw, dest, dtype, n in items:
        fast = None if lw.pscalars else _fast(lw.vectors, dest)
        if fast is None:
            rest.append((lw, dest, dtype, n))
            continue
        dev, ptrs, dptr = fast
        key = (dev, _dtype_code(dtype), " ".join(lw.tokens), len(lw.vectors), len(lw.scalars))
        groups.setdefault(key, []).append((ptrs, dptr, lw.scalars, n))
    lib = _native.lib()
    batched = 0
    for (dev, code, sig, nl, ns), probs in groups.items():
        leaves, k1 = _native.ptr_array([p for ptrs, _, _, _ in probs for p in ptrs])
        dsts, k2 = _native.ptr_array([d for _, d, _, _ in probs])
        scal, k3 = _native.double_array([c for _, _, sc, _ in probs for c in sc])
        lens = array.array("q", [n for _, _, _, n in probs])
        with _OnDevice(dev):
            _native.check(lib.salt_assign_batch(code, sig.encode(), len(probs), dsts, leaves, nl, scal, ns,
                                                lens.buffer_info()[0], _raw_stream(dev)))
        batched += len(probs)
    for lw, dest, dtype, n in rest:
        run_assign(lw, dest, dtype, n)
    return batched


def _batch_out(index: int, count: int):
    """(tensor, data pointer) of count 16-byte result slots on a device (the
    C fast path's reduce_batch)."""
    t = torch.empty(2 * count, dtype=torch.float64, device=torch.device("cuda", index))
    return t, t.data_ptr()


def batch_results(out, slots, dt, lazy):
    """Element-typed results from the 16-byte slots of `out` (one copy to
    the host unless lazy)."""
    dt = as_dtype(dt)
    if lazy:
        return [DeviceScalar(out[2 * q:2 * q + 1].view(torch.float32)[:1] if dt.itemsize == 4
                             else out[2 * q:2 * q + 1], dt) for q in slots]
    host = out.cpu().numpy()
    if dt.itemsize == 8:
        vals = host[0::2]
    else:
        vals = host.view(np.float32)[0::4]
    return [vals[q] for q in slots]


def run_reduce_batch(items, flags=0, lazy=False):
    """items: [(lowering, dtype, n)] of validated sums.  Plain-device ones
    are grouped by (device, element type, signature) and each group is one
    salt_reduce_batch call writing into one device buffer; the results then
    come back to the host in ONE copy per group (or stay on the device as
    DeviceScalars with lazy=True).  Others run one by one."""
    results = [None] * len(items)
    groups = {}
    for i, (lw, dtype, n) in enumerate(items):
        fast = None if lw.pscalars else _fast(lw.vectors, None)
        if fast is None:
            results[i] = run_reduce(lw, dtype, n, flags=flags, lazy=lazy)
            continue
        dev, ptrs, _ = fast
        key = (dev, _dtype_code(dtype), " ".join(lw.tokens), len(lw.vectors), len(lw.scalars))
        groups.setdefault(key, []).append((i, ptrs, lw.scalars, n, as_dtype(dtype)))
    lib = _native.lib()
    for (dev, code, sig, nl, ns), probs in groups.items():
        device = torch.device("cuda", dev)
        out = torch.empty(2 * len(probs), dtype=torch.float64, device=device)
        base = out.data_ptr()
        outs, k0 = _native.ptr_array([base + 16 * q for q in range(len(probs))])
        leaves, k1 = _native.ptr_array([p for _, ptrs, _, _, _ in probs for p in ptrs])
        scal, k2 = _native.double_array([c for _, _, sc, _, _ in probs for c in sc])
        lens = array.array("q", [n for _, _, _, n, _ in probs])
        with _OnDevice(dev):
            stream = _raw_stream(dev)
            ws = _workspace(dev, stream)
            _native.check(lib.salt_reduce_batch(code, sig.encode(), len(probs), leaves, nl, scal, ns,
                                                lens.buffer_info()[0], flags, outs, ws.data_ptr(),
                                                ws.numel(), stream))
        dt = probs[0][4]
        if lazy:
            for q, (i, *_rest) in enumerate(probs):
                slot = out[2 * q:2 * q + 2]
                results[i] = DeviceScalar(slot.view(torch.float32)[:1] if dt.itemsize == 4 else slot[:1], dt)
        else:
            host = out.cpu().numpy().view(np.uint8).reshape(len(probs), 16)
            for q, (i, *_rest) in enumerate(probs):
                results[i] = np.frombuffer(host[q, :dt.itemsize].tobytes(), dtype=dt)[0]
    return results


# ---------------------------------------------------------------- reduce
def _result(dt, out, host, lazy):
    if lazy:
        return DeviceScalar(out.view(torch.float32)[:1] if dt.itemsize == 4 else out, dt)
    return np.frombuffer(bytes(host)[: dt.itemsize], dtype=dt)[0]


def _device_reduce(dev, dt, call, flags, lazy, sharded=None, xcall=None):
    """call(flags, ws, wsb, out_dev, out_host, stream) -> rc on device `dev`;
    xcall(..., exchange, out_dev, out_host, stream) is the NVLink-exchange
    variant used for sharded operands when peer memory is available."""
    lib = _native.lib()
    stream = _raw_stream(dev)
    ws = _workspace(dev, stream)
    out = torch.empty(1, dtype=torch.float64, device=torch.device("cuda", dev))
    host = None if lazy else (ctypes.c_double * 2)()
    hptr = ctypes.addressof(host) if host is not None else None
    xchg = None
    # The peer exchange advances an epoch per call on the host, so it cannot
    # be baked into a CUDA graph; while capturing, the (capturable) NCCL
    # all-gather path is used instead — same bits.
    if sharded is not None and xcall is not None and not torch.cuda.is_current_stream_capturing():
        from .sharding import peer_exchange

        xchg = peer_exchange(sharded.group, torch.device("cuda", dev))
    if sharded is None:
        _native.check(call(flags, ws.data_ptr(), ws.numel(), out.data_ptr(), hptr, stream))
    elif xchg is not None:
        desc = xchg.next()
        _native.check(xcall(flags, ws.data_ptr(), ws.numel(), ctypes.addressof(desc),
                            out.data_ptr(), hptr, stream))
        if lazy:
            return DeviceScalar(out.view(torch.float32)[:1] if dt.itemsize == 4 else out, dt,
                                guard=xchg.check)
        result = _result(dt, out, host, lazy)
        xchg.check(result)  # NaN + the error word: a peer never arrived
        return result
    else:
        part = torch.empty(2, dtype=torch.float64, device=out.device)
        _native.check(call(flags | _native.SALT_PARTIAL, ws.data_ptr(), ws.numel(), part.data_ptr(),
                           None, stream))
        parts = sharded.gather_partials(part)
        _native.check(lib.salt_reduce_finish(_dtype_code(dt), parts.data_ptr(), parts.numel() // 2,
                                             flags, out.data_ptr(), hptr, stream))
    return _result(dt, out, host, lazy)


def _run_reduction(lw, dest, dt, n, flags, lazy, make_call, host_call, make_xcall=None):
    """Fast path / placement for a reduction-producing call; `host_call` runs
    it on pinned host vectors (streamed through the GPU)."""
    fast = _fast(lw.vectors, dest)
    if fast is not None:
        dev, ptrs, dptr = fast
        leaves, keep = _native.ptr_array(ptrs)
        call = make_call(leaves, dptr, n)
        if torch.cuda.current_device() == dev:
            return _device_reduce(dev, dt, call, flags, lazy)
        with _OnDevice(dev):
            return _device_reduce(dev, dt, call, flags, lazy)
    pl = Placement(lw.vectors, dest, n)
    leaves, keep = _native.ptr_array(pl.pointers)
    if pl.kind == "host":
        host = (ctypes.c_double * 2)()
        _host_call(lambda st, sb, sp: host_call(leaves, pl.n, st, sb, sp, ctypes.addressof(host),
                                                pl.dest_pointer))
        result = np.frombuffer(bytes(host)[: dt.itemsize], dtype=dt)[0]
    else:
        xcall = make_xcall(leaves, pl.dest_pointer, pl.n) if make_xcall is not None else None
        with _OnDevice(pl.device.index):
            result = _device_reduce(pl.device.index, dt, make_call(leaves, pl.dest_pointer, pl.n),
                                    flags, lazy, pl.sharded, xcall)
    pl.finish()
    _record_counts(lw, dest, n)
    return result


def run_reduce(lw, dtype, n, flags=0, lazy=False):
    if lw.pscalars:
        handled, r = run_fused(None, " ".join(lw.tokens), lw, [], dtype, n, flags, lazy)
        _device_scalars_only(handled)
        return r
    lib = _native.lib()
    dt = as_dtype(dtype)
    code = _dtype_code(dt)
    sig = " ".join(lw.tokens).encode()
    scal, keep_s = _native.double_array(lw.scalars)
    nl, ns = len(lw.vectors), len(lw.scalars)

    def make_call(leaves, _dptr, m):
        return lambda fl, ws, wsb, od, oh, st: lib.salt_reduce(
            code, sig, leaves, nl, scal, ns, m, fl, ws, wsb, od, oh, st)

    def host_call(leaves, m, st, sb, sp, out, _dptr):
        return lib.salt_reduce_host(code, sig, leaves, nl, scal, ns, m, flags, st, sb, sp, out)

    def make_xcall(leaves, _dptr, m):
        return lambda fl, ws, wsb, x, od, oh, st: lib.salt_reduce_exchange(
            code, sig, leaves, nl, scal, ns, m, fl, ws, wsb, x, od, oh, st)

    return _run_reduction(lw, None, dt, n, flags, lazy, make_call, host_call, make_xcall)


def run_assign_reduce(lwa, lwr, dest, dtype, n, flags=0, lazy=False):
    if lwa.pscalars:
        handled, r = run_fused(" ".join(lwa.tokens), " ".join(lwr.tokens), lwa, [dest], dtype, n,
                               flags, lazy)
        _device_scalars_only(handled)
        return r
    lib = _native.lib()
    dt = as_dtype(dtype)
    code = _dtype_code(dt)
    asig = " ".join(lwa.tokens).encode()
    rsig = " ".join(lwr.tokens).encode()
    scal, keep_s = _native.double_array(lwa.scalars)
    nl, ns = len(lwa.vectors), len(lwa.scalars)

    def make_call(leaves, dptr, m):
        return lambda fl, ws, wsb, od, oh, st: lib.salt_assign_reduce(
            code, asig, rsig, dptr, leaves, nl, scal, ns, m, fl, ws, wsb, od, oh, st)

    def host_call(leaves, m, st, sb, sp, out, dptr):
        return lib.salt_assign_reduce_host(code, asig, rsig, dptr, leaves, nl, scal, ns, m, flags,
                                           st, sb, sp, out)

    def make_xcall(leaves, dptr, m):
        return lambda fl, ws, wsb, x, od, oh, st: lib.salt_assign_reduce_exchange(
            code, asig, rsig, dptr, leaves, nl, scal, ns, m, fl, ws, wsb, x, od, oh, st)

    return _run_reduction(lwa, dest, dt, n, flags, lazy, make_call, host_call, make_xcall)


def run_fused(asig, rsig, lw, dests, dtype, n, flags=0, lazy=False):
    """salt_fused: several assignment roots (asig, ' ; '-separated, or None)
    and/or a reduction (rsig or None), with device-scalar operands
    (lw.pscalars).  Returns (handled, result): not handled unless every leaf
    and destination is a plain device DenseVector on one device."""
    fast = _fast(list(lw.vectors) + list(dests), None)
    sharded = None
    if fast is None:
        # Sharded operands: every rank runs the same kernel on its blocks;
        # a reduction's per-rank partials meet in a 16-byte all-gather and a
        # fixed-order finish (same bits on every rank), so device scalars
        # computed from it stay identical across ranks.
        shards = _sharded_operands(list(lw.vectors) + list(dests))
        if shards is None:
            return False, None
        sharded = shards[0]
        dev = sharded.local.device.index
        ptrs = [s.local.tensor.data_ptr() for s in shards]
        n = len(sharded.local)
    else:
        dev, ptrs, _ = fast
    for ds in lw.pscalars:
        if ds.device.index != dev:
            raise ValueError("a device scalar must live on the vectors' device")
    nl = len(lw.vectors)
    leaves, keep_l = _native.ptr_array(ptrs[:nl])
    dsts, keep_d = _native.ptr_array(ptrs[nl:])
    raw, host, prog = _scalar_program(lw.pscalars, list(lw.scalars))
    scal, keep_s = _native.double_array(host)
    pscal, keep_p = _native.ptr_array([ds.tensor.data_ptr() for ds in raw])
    dt = as_dtype(dtype)
    code = _dtype_code(dt)
    lib = _native.lib()
    a = asig.encode() if asig is not None else None
    r = rsig.encode() if rsig is not None else None
    np_ = len(raw)
    sp = prog.encode() if prog else None
    with _OnDevice(dev):
        if rsig is None:
            _native.check(lib.salt_fused_prog(code, a, None, dsts, len(dests), leaves, nl, scal,
                                              len(host), pscal, np_, sp, n, 0, None, 0, None, None,
                                              _raw_stream(dev)))
            return True, None

        def call(fl, ws, wsb, od, oh, st):
            return lib.salt_fused_prog(code, a, r, dsts, len(dests), leaves, nl, scal, len(host),
                                       pscal, np_, sp, n, fl, ws, wsb, od, oh, st)

        def xcall(fl, ws, wsb, x, od, oh, st):
            return lib.salt_fused_exchange_prog(code, a, r, dsts, len(dests), leaves, nl, scal,
                                                len(host), pscal, np_, sp, n, fl, ws, wsb, x, od,
                                                oh, st)

        return True, _device_reduce(dev, dt, call, flags, lazy, sharded,
                                    xcall if sharded is not None else None)


def _scalar_program(pscalars, host):
    """(raw device scalars, host scalars, program text or None) for the
    tree's device-scalar operands P0..P(k-1).  Without a lazy operand the raw
    list IS pscalars and there is no program.  Otherwise every P<k> gets a
    postfix program over the raw (materialised) device scalars "p<i>" and
    host scalars "S<j>" (appended to `host`), evaluated once per thread in
    the kernel prologue (csrc/salt_expr.cuh load_pscalars)."""
    budget = DeviceScalar.MAX_PROGRAM_OPS
    if not any(ds.lazy and ds.program_size() <= budget for ds in pscalars):
        return list(pscalars), host, None  # (an oversized lazy scalar materialises when read)
    for ds in pscalars:
        ds.check_operands()
    raw, raw_ids, toks = [], {}, []

    def emit(x):
        if isinstance(x, DeviceScalar) and (not x.lazy or x.program_size() > budget):
            i = raw_ids.get(id(x))
            if i is None:
                if len(raw) == _native.SALT_MAX_PSCALARS:
                    raise _ProgramTooLarge
                i = raw_ids[id(x)] = len(raw)
                raw.append(x)
            toks.append(f"p{i}")
        elif isinstance(x, DeviceScalar):
            op, *args = x._expr
            for arg in args:
                emit(arg)
            toks.append(op)
        else:
            if len(host) == _native.SALT_MAX_SCALARS:
                raise _ProgramTooLarge
            toks.append(f"S{len(host)}")
            host.append(float(x))

    n0 = len(host)
    try:
        for k, ds in enumerate(pscalars):
            emit(ds)
            toks.append(f"={k}")
        if len(toks) > 32:
            raise _ProgramTooLarge
    except _ProgramTooLarge:  # materialise everything: one raw pointer per operand
        del host[n0:]
        return list(pscalars), host, None
    return raw, host, " ".join(toks)


class _ProgramTooLarge(Exception):
    pass


def _sharded_operands(vectors):
    """The ShardedVectors behind `vectors` if ALL are sharded, share one
    partition and live on a CUDA device; else None."""
    from .sharding import ShardedVector

    shards = [_shard_of(v) for v in vectors]
    if not shards or not all(isinstance(s, ShardedVector) for s in shards):
        return None
    first = shards[0]
    if first.local.device.type != "cuda":
        return None
    for s in shards[1:]:
        if not first.same_partition(s):
            raise ValueError("sharded vectors in one expression must share a partition")
    return shards


def _device_scalars_only(handled):
    if not handled:
        raise TypeError("trees with device-scalar operands need plain device DenseVector "
                        "operands on one device")
