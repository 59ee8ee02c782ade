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

Operands are resolved to their storage first: DenseVector itself, the inner
vector of a CountingVector, the local block of a ShardedVector, or — for any
other duck-typed vector (expressions.py:68-69) — a temporary device copy made
through its read_block/write_block protocol.
"""

import ctypes
import threading

import numpy as np
import torch

from . import _native
from .lanes import as_dtype
from .vectors import DenseVector, DeviceScalar

__all__ = ["run_assign", "run_reduce", "run_assign_reduce", "Placement"]

_ws_lock = threading.Lock()
_workspaces = {}
_host_state = {}
_HOST_STAGING_BYTES = 768 << 20


def _dtype_code(dt: np.dtype) -> int:
    return _native.SALT_F32 if as_dtype(dt).itemsize == 4 else _native.SALT_F64


def _unwrap(vec):
    """Storage DenseVector behind `vec` (or None for a foreign duck vector)."""
    seen = 0
    while not isinstance(vec, DenseVector):
        inner = getattr(vec, "inner", None)
        if inner is None or seen > 8:
            return None
        vec, seen = inner, seen + 1
    return vec


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

    def finish(self):
        if self.staged_dest is not None:
            v, staged = self.staged_dest
            v.write_block(0, len(v), staged.to_array())


def _shard_of(v):
    from .sharding import ShardedVector

    seen = 0
    while not isinstance(v, ShardedVector) and seen < 8:
        inner = getattr(v, "inner", None)
        if inner is None:
            return v
        v, seen = inner, seen + 1
    return v


def _require_cuda() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError(
            "no CUDA device: paper_1109_1264_b200 evaluates expressions on the GPU only "
            "(there is no CPU evaluation path)"
        )
    return torch.device("cuda", torch.cuda.current_device())


def _workspace(device: torch.device, stream_ptr: int) -> torch.Tensor:
    key = (device.index, stream_ptr)
    ws = _workspaces.get(key)
    if ws is None:
        with _ws_lock:
            ws = _workspaces.get(key)
            if ws is None:
                nbytes = _native.lib().salt_reduce_workspace_bytes()
                ws = torch.zeros(nbytes, dtype=torch.uint8, device=device)
                _workspaces[key] = ws
    return ws


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


def _pointers(storage):
    return [s.tensor.data_ptr() for s in storage]


def _record_counts(lw, dest, n):
    """CountingVector bookkeeping: each leaf OCCURRENCE reads n elements and
    the destination is written n times (reference semantics, test_engine.py
    :468-485), even though the fused kernel loads a repeated leaf once."""
    for vec, occ in zip(lw.vectors, lw.occurrences):
        if hasattr(vec, "read_count"):
            vec.read_count += occ * n
    if dest is not None and hasattr(dest, "write_count"):
        dest.write_count += n


def run_assign(lw, dest, dtype, n):
    pl = Placement(lw.vectors, dest, n)
    code = _dtype_code(dtype)
    lib = _native.lib()
    sig = " ".join(lw.tokens).encode()
    leaves, _keep = _native.ptr_array(_pointers(pl.leaves))
    scal, _keep2 = _native.double_array(lw.scalars)
    if pl.kind == "host":
        if pl.n == 0:
            return
        dev = _require_cuda()
        lock, staging, streams = _host_resources(dev)
        with lock, torch.cuda.device(dev):
            sptrs, _keep3 = _native.ptr_array([s.cuda_stream for s in streams])
            torch.cuda.current_stream(dev).synchronize()
            _native.check(
                lib.salt_assign_host(
                    code, sig, pl.dest.tensor.data_ptr(), leaves, len(pl.leaves), scal,
                    len(lw.scalars), pl.n, staging.data_ptr(), staging.numel(), sptrs,
                )
            )
    else:
        with torch.cuda.device(pl.device):
            stream = torch.cuda.current_stream(pl.device).cuda_stream
            _native.check(
                lib.salt_assign(
                    code, sig, pl.dest.tensor.data_ptr(), leaves, len(pl.leaves), scal,
                    len(lw.scalars), pl.n, stream,
                )
            )
    pl.finish()
    _record_counts(lw, dest, n)


def _reduce_common(pl, dtype, call_partial, flags, lazy):
    """Run a device reduction; handles the sharded all-gather + finish."""
    code = _dtype_code(dtype)
    lib = _native.lib()
    dt = as_dtype(dtype)
    with torch.cuda.device(pl.device):
        stream = torch.cuda.current_stream(pl.device).cuda_stream
        ws = _workspace(pl.device, stream)
        if pl.sharded is not None:
            part = torch.empty(2, dtype=torch.float64, device=pl.device)
            _native.check(
                call_partial(flags | _native.SALT_PARTIAL, ws, part.data_ptr(), None, stream)
            )
            parts = pl.sharded.gather_partials(part)
            out = torch.empty(1, dtype=torch.float64, device=pl.device)
            host = None if lazy else (ctypes.c_double * 2)()
            _native.check(
                lib.salt_reduce_finish(
                    code, parts.data_ptr(), parts.numel() // 2, flags, out.data_ptr(),
                    ctypes.addressof(host) if host is not None else None, stream,
                )
            )
        else:
            out = torch.empty(1, dtype=torch.float64, device=pl.device)
            host = None if lazy else (ctypes.c_double * 2)()
            _native.check(
                call_partial(
                    flags, ws, out.data_ptr(), ctypes.addressof(host) if host is not None else None,
                    stream,
                )
            )
    if lazy:
        view = out.view(torch.float32)[:1] if dt.itemsize == 4 else out
        return DeviceScalar(view, dt)
    raw = bytes(host)[: dt.itemsize]
    return np.frombuffer(raw, dtype=dt)[0]


def run_reduce(lw, dtype, n, flags=0, lazy=False):
    pl = Placement(lw.vectors, None, n)
    code = _dtype_code(dtype)
    lib = _native.lib()
    sig = " ".join(lw.tokens).encode()
    leaves, _keep = _native.ptr_array(_pointers(pl.leaves))
    scal, _keep2 = _native.double_array(lw.scalars)
    if pl.kind == "host":
        dev = _require_cuda()
        lock, staging, streams = _host_resources(dev)
        host = (ctypes.c_double * 2)()
        with lock, torch.cuda.device(dev):
            sptrs, _keep3 = _native.ptr_array([s.cuda_stream for s in streams])
            torch.cuda.current_stream(dev).synchronize()
            _native.check(
                lib.salt_reduce_host(
                    code, sig, leaves, len(pl.leaves), scal, len(lw.scalars), pl.n, flags,
                    staging.data_ptr(), staging.numel(), sptrs, ctypes.addressof(host),
                )
            )
        _record_counts(lw, None, n)
        dt = as_dtype(dtype)
        return np.frombuffer(bytes(host)[: dt.itemsize], dtype=dt)[0]

    def call(fl, ws, out_dev, out_host, stream):
        return lib.salt_reduce(
            code, sig, leaves, len(pl.leaves), scal, len(lw.scalars), pl.n, fl, ws.data_ptr(),
            ws.numel(), out_dev, out_host, stream,
        )

    result = _reduce_common(pl, dtype, call, flags, lazy)
    _record_counts(lw, None, n)
    return result


def run_assign_reduce(lwa, lwr, dest, dtype, n, flags=0, lazy=False):
    pl = Placement(lwa.vectors, dest, n)
    if pl.kind == "host":
        raise TypeError("fused assign+reduce needs device-resident vectors")
    code = _dtype_code(dtype)
    lib = _native.lib()
    asig = " ".join(lwa.tokens).encode()
    rsig = " ".join(lwr.tokens).encode()
    leaves, _keep = _native.ptr_array(_pointers(pl.leaves))
    scal, _keep2 = _native.double_array(lwa.scalars)
    dst = pl.dest.tensor.data_ptr()

    def call(fl, ws, out_dev, out_host, stream):
        return lib.salt_assign_reduce(
            code, asig, rsig, dst, leaves, len(pl.leaves), scal, len(lwa.scalars), pl.n, fl,
            ws.data_ptr(), ws.numel(), out_dev, out_host, stream,
        )

    result = _reduce_common(pl, dtype, call, flags, lazy)
    pl.finish()
    _record_counts(lwa, dest, n)
    return result
