"""ctypes wrapper of salt_oracle.c (TEST INFRASTRUCTURE ONLY).

oracle_assign / oracle_reduce take NumPy arrays and the same postfix
signatures as libsalt.so.  The library is built by `make -C oracle`
(also run by __graft_entry__.build()).
"""

import ctypes
from pathlib import Path

import numpy as np

__all__ = ["available", "assign", "reduce", "reduce_exact", "LIB_PATH"]

LIB_PATH = Path(__file__).with_name("_build") / "liboracle.so"
_DT = {"f32": np.float32, "f64": np.float64}
_lib = None


def _load():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise RuntimeError(f"{LIB_PATH} missing: run `make -C oracle`")
        lib = ctypes.CDLL(str(LIB_PATH))
        vp, vpp = ctypes.c_void_p, ctypes.POINTER(ctypes.c_void_p)
        dp = ctypes.POINTER(ctypes.c_double)
        lib.oracle_assign.argtypes = [ctypes.c_int, ctypes.c_char_p, vp, vpp, ctypes.c_int, dp,
                                      ctypes.c_int, ctypes.c_int64, ctypes.c_int]
        lib.oracle_assign.restype = ctypes.c_int
        lib.oracle_reduce.argtypes = [ctypes.c_int, ctypes.c_char_p, ctypes.c_char_p, vp, vpp,
                                      ctypes.c_int, dp, ctypes.c_int, ctypes.c_int64, ctypes.c_int,
                                      ctypes.c_int, ctypes.c_int, vp]
        lib.oracle_reduce.restype = ctypes.c_int
        lib.oracle_reduce_exact.argtypes = [ctypes.c_int, ctypes.c_char_p, ctypes.c_char_p, vpp,
                                            ctypes.c_int, dp, ctypes.c_int, ctypes.c_int64,
                                            ctypes.c_int, dp]
        lib.oracle_reduce_exact.restype = ctypes.c_int
        _lib = lib
    return _lib


def available() -> bool:
    return LIB_PATH.exists()


def _args(leaves, scalars):
    ptrs = (ctypes.c_void_p * max(1, len(leaves)))(*[a.ctypes.data for a in leaves])
    sc = (ctypes.c_double * max(1, len(scalars)))(*[float(s) for s in scalars])
    return ctypes.cast(ptrs, ctypes.POINTER(ctypes.c_void_p)), ctypes.cast(sc, ctypes.POINTER(ctypes.c_double)), (ptrs, sc)


def assign(sig, dst, leaves, scalars, threads=1):
    """dst[:] = tree(leaves, scalars) in the element type of dst."""
    code = 0 if dst.dtype == np.float32 else 1
    leaves = [np.ascontiguousarray(a, dtype=dst.dtype) if a is not dst else a for a in leaves]
    lp, sp, keep = _args(leaves, scalars)
    rc = _load().oracle_assign(code, sig.encode(), dst.ctypes.data, lp, len(leaves), sp,
                               len(scalars), dst.shape[0], threads)
    if rc:
        raise ValueError(f"oracle_assign failed ({rc}) for {sig!r}")
    return dst


def reduce(sig, leaves, scalars, dtype, unroll, width, threads=1, assign_sig=None, dst=None):
    """Reference-engine-order reduction (bit-exact for threads=1).  With
    assign_sig, dst is assigned first and `D` in sig reads it (fused)."""
    dt = np.dtype(_DT.get(dtype, dtype) if isinstance(dtype, str) else dtype)
    code = 0 if dt == np.float32 else 1
    leaves = [np.ascontiguousarray(a, dtype=dt) if a is not dst else a for a in leaves]
    lp, sp, keep = _args(leaves, scalars)
    out = np.zeros(1, dtype=dt)
    n = leaves[0].shape[0] if leaves else (dst.shape[0] if dst is not None else 0)
    rc = _load().oracle_reduce(code, assign_sig.encode() if assign_sig else None, sig.encode(),
                               dst.ctypes.data if dst is not None else None, lp, len(leaves), sp,
                               len(scalars), n, unroll, width, threads, out.ctypes.data)
    if rc:
        raise ValueError(f"oracle_reduce failed ({rc}) for {sig!r}")
    return out[0]


def reduce_exact(sig, leaves, scalars, dtype, threads=8, assign_sig=None):
    """Sum of the tree's element-typed values accumulated in binary128
    (near-exact); returns a Python float.  With assign_sig, `D` in sig reads
    the assign tree's value (nothing is stored)."""
    dt = np.dtype(_DT.get(dtype, dtype) if isinstance(dtype, str) else dtype)
    code = 0 if dt == np.float32 else 1
    leaves = [np.ascontiguousarray(a, dtype=dt) for a in leaves]
    lp, sp, keep = _args(leaves, scalars)
    out = ctypes.c_double(0.0)
    n = leaves[0].shape[0] if leaves else 0
    rc = _load().oracle_reduce_exact(code, assign_sig.encode() if assign_sig else None,
                                     sig.encode(), lp, len(leaves), sp, len(scalars), n, threads,
                                     ctypes.byref(out))
    if rc:
        raise ValueError(f"oracle_reduce_exact failed ({rc}) for {sig!r}")
    return out.value
