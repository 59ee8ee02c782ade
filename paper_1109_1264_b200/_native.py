"""ctypes binding of libsalt.so (the C ABI declared in include/salt.h).

This module is the only place Python talks to native code.  There is no CPU
fallback: if the library is missing or a CUDA call fails, the error is raised
here (RuntimeError with the library's thread-local message), mirroring how the
reference surfaces failures as exceptions (error
conventions).
"""

import array
import ctypes
import os
import threading
from pathlib import Path

__all__ = [
    "lib",
    "check",
    "SALT_F32",
    "SALT_F64",
    "SALT_SQRT",
    "SALT_PARTIAL",
    "LIB_PATH",
    "HEADER_SYMBOLS",
]

SALT_WORKSPACE_TICKET_BYTES = 1065216
SALT_MAX_LEAVES = 16
SALT_MAX_SCALARS = 32
SALT_MAX_ROOTS = 4
SALT_MAX_PSCALARS = 8
SALT_F32 = 0
SALT_F64 = 1
SALT_SQRT = 1
SALT_PARTIAL = 2

LIB_PATH = Path(os.environ.get("SALT_LIB", Path(__file__).with_name("libsalt.so")))

# Every function include/salt.h declares (tests check the .so exports them all).
HEADER_SYMBOLS = (
    "salt_assign",
    "salt_reduce",
    "salt_assign_reduce",
    "salt_fused",
    "salt_fused_prog",
    "salt_assign_batch",
    "salt_reduce_batch",
    "salt_reduce_finish",
    "salt_assign_host",
    "salt_reduce_host",
    "salt_assign_reduce_host",
    "salt_reduce_workspace_bytes",
    "salt_capture_id",
    "salt_set_trace",
    "salt_result_enqueue",
    "salt_result_slot",
    "salt_stream_synchronize",
    "salt_reduce_exchange",
    "salt_assign_reduce_exchange",
    "salt_fused_exchange",
    "salt_fused_exchange_prog",
    "salt_exchange_emulate",
    "salt_allreduce_sum",
    "salt_allreduce_sum_flags",
    "salt_nccl_comm_init_all",
    "salt_nccl_comm_destroy",
    "salt_group_create",
    "salt_group_destroy",
    "salt_group_size",
    "salt_group_fused",
    "salt_group_issue_times",
    "salt_group_fused_exchange",
    "salt_enable_peer_access",
    "salt_signature_kind",
    "salt_prepare",
    "salt_set_force_jit",
    "salt_set_force_interp",
    "salt_interp_launch_count",
    "salt_set_jit_async",
    "salt_jit_wait",
    "salt_launch_count",
    "salt_last_error",
    "salt_abi_version",
)

_c_int = ctypes.c_int
_c_i64 = ctypes.c_int64
_c_size = ctypes.c_size_t
_c_vp = ctypes.c_void_p
_c_str = ctypes.c_char_p
# Pointer arrays / scalar arrays are passed as raw addresses (array.array
# buffers): building ctypes arrays per call costs several microseconds.
_c_vpp = ctypes.c_void_p
_c_dp = ctypes.c_void_p

_SIGNATURES = {
    "salt_assign": (_c_int, [_c_int, _c_str, _c_vp, _c_vpp, _c_int, _c_dp, _c_int, _c_i64, _c_vp]),
    "salt_reduce": (
        _c_int,
        [_c_int, _c_str, _c_vpp, _c_int, _c_dp, _c_int, _c_i64, _c_int, _c_vp, _c_size, _c_vp, _c_vp, _c_vp],
    ),
    "salt_assign_reduce": (
        _c_int,
        [_c_int, _c_str, _c_str, _c_vp, _c_vpp, _c_int, _c_dp, _c_int, _c_i64, _c_int, _c_vp, _c_size,
         _c_vp, _c_vp, _c_vp],
    ),
    "salt_fused": (
        _c_int,
        [_c_int, _c_str, _c_str, _c_vpp, _c_int, _c_vpp, _c_int, _c_dp, _c_int, _c_vpp, _c_int,
         _c_i64, _c_int, _c_vp, _c_size, _c_vp, _c_vp, _c_vp],
    ),
    "salt_fused_prog": (
        _c_int,
        [_c_int, _c_str, _c_str, _c_vpp, _c_int, _c_vpp, _c_int, _c_dp, _c_int, _c_vpp, _c_int, _c_str,
         _c_i64, _c_int, _c_vp, _c_size, _c_vp, _c_vp, _c_vp],
    ),
    "salt_fused_exchange_prog": (
        _c_int,
        [_c_int, _c_str, _c_str, _c_vpp, _c_int, _c_vpp, _c_int, _c_dp, _c_int, _c_vpp, _c_int, _c_str,
         _c_i64, _c_int, _c_vp, _c_size, _c_vp, _c_vp, _c_vp, _c_vp],
    ),
    "salt_reduce_finish": (_c_int, [_c_int, _c_vp, _c_int, _c_int, _c_vp, _c_vp, _c_vp]),
    "salt_assign_batch": (_c_int, [_c_int, _c_str, _c_int, _c_vpp, _c_vpp, _c_int, _c_dp, _c_int, _c_vp, _c_vp]),
    "salt_reduce_batch": (_c_int, [_c_int, _c_str, _c_int, _c_vpp, _c_int, _c_dp, _c_int, _c_vp, _c_int, _c_vpp,
                                   _c_vp, _c_size, _c_vp]),
    "salt_assign_host": (
        _c_int, [_c_int, _c_str, _c_vp, _c_vpp, _c_int, _c_dp, _c_int, _c_i64, _c_vp, _c_size, _c_vpp]
    ),
    "salt_reduce_host": (
        _c_int,
        [_c_int, _c_str, _c_vpp, _c_int, _c_dp, _c_int, _c_i64, _c_int, _c_vp, _c_size, _c_vpp, _c_vp],
    ),
    "salt_assign_reduce_host": (
        _c_int,
        [_c_int, _c_str, _c_str, _c_vp, _c_vpp, _c_int, _c_dp, _c_int, _c_i64, _c_int, _c_vp, _c_size,
         _c_vpp, _c_vp],
    ),
    "salt_reduce_workspace_bytes": (_c_size, []),
    "salt_capture_id": (ctypes.c_uint64, [_c_vp]),
    "salt_set_trace": (_c_int, [_c_vp, _c_i64]),
    "salt_result_enqueue": (_c_int, [_c_vp, _c_size, _c_vp, _c_vp]),
    "salt_result_slot": (_c_int, [_c_vp]),
    "salt_stream_synchronize": (_c_int, [_c_vp]),
    "salt_reduce_exchange": (
        _c_int,
        [_c_int, _c_str, _c_vpp, _c_int, _c_dp, _c_int, _c_i64, _c_int, _c_vp, _c_size, _c_vp, _c_vp,
         _c_vp, _c_vp],
    ),
    "salt_assign_reduce_exchange": (
        _c_int,
        [_c_int, _c_str, _c_str, _c_vp, _c_vpp, _c_int, _c_dp, _c_int, _c_i64, _c_int, _c_vp, _c_size,
         _c_vp, _c_vp, _c_vp, _c_vp],
    ),
    "salt_fused_exchange": (
        _c_int,
        [_c_int, _c_str, _c_str, _c_vpp, _c_int, _c_vpp, _c_int, _c_dp, _c_int, _c_vpp, _c_int,
         _c_i64, _c_int, _c_vp, _c_size, _c_vp, _c_vp, _c_vp, _c_vp],
    ),
    "salt_exchange_emulate": (_c_int, [_c_int, _c_int, ctypes.c_uint64, _c_vp, _c_vp, _c_vp, _c_vp]),
    "salt_allreduce_sum": (_c_int, [_c_vpp, _c_int, _c_int, _c_vpp, _c_vpp]),
    "salt_allreduce_sum_flags": (_c_int, [_c_vpp, _c_int, _c_int, _c_vpp, _c_vpp, _c_int]),
    "salt_nccl_comm_init_all": (_c_int, [_c_int, _c_vp, _c_vpp]),
    "salt_nccl_comm_destroy": (_c_int, [_c_int, _c_vpp]),
    "salt_group_create": (_c_int, [_c_int, _c_vp, _c_vp]),
    "salt_group_destroy": (_c_int, [_c_vp]),
    "salt_group_size": (_c_int, [_c_vp]),
    "salt_group_fused": (
        _c_int,
        [_c_vp, _c_int, _c_str, _c_str, _c_vpp, _c_int, _c_vpp, _c_int, _c_dp, _c_int, _c_vpp, _c_int,
         _c_vp, _c_int, _c_vpp, _c_size, _c_vpp, _c_vpp],
    ),
    "salt_group_issue_times": (_c_int, [_c_vp, _c_vp, _c_vp]),
    "salt_group_fused_exchange": (
        _c_int,
        [_c_vp, _c_int, _c_str, _c_str, _c_vpp, _c_int, _c_vpp, _c_int, _c_dp, _c_int, _c_vpp, _c_int,
         _c_vp, _c_int, _c_vpp, _c_size, _c_vp, _c_vpp, _c_vpp],
    ),
    "salt_enable_peer_access": (_c_int, [_c_int, _c_vp]),
    "salt_signature_kind": (_c_int, [_c_int, _c_str, _c_str, _c_int]),
    "salt_prepare": (_c_int, [_c_int, _c_str, _c_str, _c_int]),
    "salt_set_force_jit": (None, [_c_int]),
    "salt_set_force_interp": (None, [_c_int]),
    "salt_interp_launch_count": (ctypes.c_uint64, []),
    "salt_set_jit_async": (None, [_c_int]),
    "salt_jit_wait": (_c_int, []),
    "salt_launch_count": (ctypes.c_uint64, []),
    "salt_last_error": (_c_str, []),
    "salt_abi_version": (_c_int, []),
}

XCHG_MAX_RANKS = 8
XCHG_BUFFER_BYTES = 512


class Exchange(ctypes.Structure):
    """salt_exchange (include/salt.h): NVLink peer-memory exchange descriptor."""

    _fields_ = [
        ("rank", ctypes.c_int32),
        ("world", ctypes.c_int32),
        ("epoch", ctypes.c_uint64),
        ("slots", ctypes.c_void_p * XCHG_MAX_RANKS),
        ("flags", ctypes.c_void_p * XCHG_MAX_RANKS),
        ("timeout_ns", ctypes.c_uint64),
        ("error", ctypes.c_void_p),
    ]


_lock = threading.RLock()
_lib = None


def lib() -> ctypes.CDLL:
    """Load libsalt.so once; raise loudly if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not LIB_PATH.exists():
                raise RuntimeError(
                    f"libsalt.so not found at {LIB_PATH}; build it with "
                    "`python -c 'import __graft_entry__ as g; g.build()'` "
                    "(there is no CPU fallback)"
                )
            handle = ctypes.CDLL(str(LIB_PATH))
            for name, (res, args) in _SIGNATURES.items():
                fn = getattr(handle, name)
                fn.restype = res
                fn.argtypes = args
            if handle.salt_abi_version() != 1:
                raise RuntimeError("libsalt.so ABI version mismatch; rebuild it")
            _lib = handle
    return _lib


_fast = None
_fast_tried = False


def fastpath():
    """The C host fast path (csrc/fastpath.c) bound to this libsalt instance,
    or None if the extension was not built (the Python path then runs)."""
    global _fast, _fast_tried
    if _fast_tried:
        return _fast
    with _lock:
        if not _fast_tried:
            try:
                import torch

                from . import _fastpath, runtime
                from .expressions import AddNode, Leaf, MulNode, ScaleNode, SubNode
                from .vectors import DenseVector, DeviceScalar
                import numpy as np

                h = lib()
                addr = lambda f: ctypes.cast(f, ctypes.c_void_p).value  # noqa: E731
                _fastpath.init(
                    addr(h.salt_assign), addr(h.salt_reduce), addr(h.salt_assign_reduce),
                    addr(h.salt_fused), addr(h.salt_last_error), h.salt_reduce_workspace_bytes(),
                    Leaf, AddNode, SubNode, MulNode, ScaleNode, DenseVector, DeviceScalar,
                    # raw C getters: CUDA is initialised once a device vector exists
                    torch._C._cuda_getCurrentRawStream, torch._C._cuda_getDevice,
                    runtime._workspace, np.float32, np.float64, runtime._lazy_out,
                    addr(h.salt_assign_batch), addr(h.salt_reduce_batch), runtime._batch_out,
                    addr(h.salt_result_enqueue), addr(h.salt_stream_synchronize),
                    addr(h.salt_fused_prog), addr(h.salt_result_slot),
                )
                _fast = _fastpath
            except (ImportError, AttributeError):
                _fast = None
            _fast_tried = True
    return _fast


def check(rc: int) -> None:
    if rc != 0:
        msg = lib().salt_last_error()
        raise RuntimeError(f"libsalt error {rc}: {msg.decode() if msg else 'unknown'}")


_EMPTY_Q = array.array("Q", [0])
_EMPTY_D = array.array("d", [0.0])


def i64_array(values):
    """(address, keep-alive) of an int64 array holding `values`."""
    arr = array.array("q", values) if values else array.array("q", [0])
    return arr.buffer_info()[0], arr


def ptr_array(ptrs):
    """(address, keep-alive) of a uint64 array holding `ptrs`."""
    arr = array.array("Q", ptrs) if ptrs else _EMPTY_Q
    return arr.buffer_info()[0], arr


def double_array(values):
    """(address, keep-alive) of a float64 array holding `values`."""
    arr = array.array("d", values) if values else _EMPTY_D
    return arr.buffer_info()[0], arr
